import sys, json, time
sys.path.insert(0, '/root/repo')
from oracle import port
from paper_2405_16256_b200 import configs, abi
name = sys.argv[1]; pps = [int(x) for x in sys.argv[2].split(",")]
cfg = configs.with_pp(configs.config(name, full=True), pps)
P = abi.Problem(cfg)
out = open(f"/tmp/stats/{name}_{sys.argv[2].replace(',','_')}.jsonl", "w")
def cb(li):
    out.write(json.dumps([li.task, li.pp, li.dp, li.B, li.M, list(li.tp)[:2], li.exhaustive, li.hill_steps, li.evaluated, li.simulated, li.pruned]) + "\n")
t0 = time.time()
st, res = port.search(P, cb)
out.write(json.dumps({"done": True, "wall": time.time()-t0, "sim": res.candidates_simulated, "pruned": res.candidates_pruned, "best": res.best_time_s, "pp": res.best_pp}) + "\n")
out.close()
