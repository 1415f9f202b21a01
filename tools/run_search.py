"""Dev tool: one search of a named config on cuda:0 (for ncu / timing)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_16256_b200 import configs, abi, planner
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
full = (sys.argv[2] if len(sys.argv) > 2 else "full") == "full"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if ":" in name and name.startswith("C3"):
    base, pps = name.split(":")
    cfg = configs.with_pp(configs.config(base, full=full), [int(x) for x in pps.split(",")])
else:
    cfg = configs.config(name, full=full)
shard = os.environ.get("RUN_SHARD")  # "r/n": one shard of an n-GPU sweep on this GPU
for _ in range(reps):
    if shard:
        r, n = (int(x) for x in shard.split("/"))
        eng = planner.Engine(0)
        t0 = time.time(); res = eng.search_shard(abi.Problem(cfg), r, n); t1 = time.time()
        print(json.dumps({"cfg": name, "shard": shard, "wall_s": t1 - t0, "dev_ms": res.device_ms,
                          "sim": res.candidates_simulated}), flush=True)
        continue
    t0 = time.time(); o = planner.search(cfg); t1 = time.time()
    print(json.dumps({"cfg": name, "wall_s": t1 - t0, "dev_ms": o.device_ms, "sim": o.candidates_simulated,
                      "pruned": o.candidates_pruned, "t": o.iteration_time_s, "launches": o.gpu_launches,
                      "ops": o.raw.eval_fp64_ops}), flush=True)
