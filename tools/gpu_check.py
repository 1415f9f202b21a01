"""Dev check: GPU search vs the C oracle on small configs, plus timings."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port
from paper_2405_16256_b200 import configs, abi, planner

def run(name, cfg, check=True):
    P = abi.Problem(cfg)
    eng = planner.engine(0)
    t0 = time.time(); r = eng.search_shard(P); t1 = time.time()
    line = {"cfg": name, "gpu_s": round(t1 - t0, 4), "dev_ms": round(r.device_ms, 2), "sim": r.candidates_simulated,
            "pruned": r.candidates_pruned, "time": r.best_time_s, "launches": r.gpu_launches,
            "enc": abi.encode_plan(P.group_names, r.best_plan)}
    if check:
        t0 = time.time(); st, o = port.search(P); t1 = time.time()
        line["oracle_s"] = round(t1 - t0, 3)
        line["match"] = (o.best_time_s == r.best_time_s and o.candidates_simulated == r.candidates_simulated and
                         o.candidates_pruned == r.candidates_pruned and
                         abi.encode_plan(P.group_names, o.best_plan) == line["enc"])
        if not line["match"]:
            line["oracle"] = [o.candidates_simulated, o.candidates_pruned, o.best_time_s, abi.encode_plan(P.group_names, o.best_plan)]
    print(json.dumps(line), flush=True)

which = sys.argv[1] if len(sys.argv) > 1 else "small"
if which == "small":
    for n in ["C0", "C1", "C2u", "C2"]:
        run(n, configs.config(n, full=True))
    run("C3pp12", configs.with_pp(configs.config("C3", full=True), [12]))
    run("C3pp24", configs.with_pp(configs.config("C3", full=True), [24]))
    c = configs.config("C5"); c["planner"]["pipeline_degrees"] = [3]; c["planner"]["micro_batch_candidates"] = [8]
    run("C5pp3B8", c)
if which in ("small", "c3"):
    for i in range(2):
        run("C3full", configs.config("C3", full=True), check=False)
