"""Dev tool: the C3 full sweep as N shards run one after another on cuda:0
(what each rank of an N-GPU run computes): per-shard device ms (an estimate
of the N-GPU rank times without the NVLink/NCCL part) and the exact
reduction checked against the unsharded search.
usage: python tools/shard_sweep.py N [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_16256_b200 import abi, configs, planner

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = abi.Problem(configs.config("C3", full=True))
eng = planner.Engine(0)
whole = eng.search_shard(p)
for _ in range(reps):
    parts = [eng.search_shard(p, s, n) for s in range(n)]
    ms = [round(r.device_ms, 1) for r in parts]
    red = planner.reduce_results(p, parts)
    ok = (red.best_time_s == whole.best_time_s and red.candidates_simulated == whole.candidates_simulated
          and red.candidates_pruned == whole.candidates_pruned
          and abi.encode_plan(p.group_names, red.best_plan) == abi.encode_plan(p.group_names, whole.best_plan))
    print(json.dumps({"shards": n, "device_ms": ms, "max_ms": max(ms), "whole_ms": round(whole.device_ms, 1),
                      "reduction_equal": ok}), flush=True)
