"""Dev tool: repeat the random-instance parity searches on the GPU to shake
out scheduling races (the climb kernel's watchdog reports ring counters)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2405_16256_b200 import abi, planner
import instances
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = planner.engine(0)
n = bad = 0
t0 = time.time()
import random
for rep in range(reps):
    rng = random.Random(99 + rep)
    for k in range(80):
        docs = instances.random_instance(rng, k)
        for full in (True, False):
            d = json.loads(json.dumps(docs))
            d["planner"]["time_bound_pruning"] = not full
            try:
                eng.search_shard(abi.Problem(d))
            except abi.InfeasibleError:
                pass
            except Exception as e:
                bad += 1
                print("rep", rep, "k", k, "full", full, "ERR", e, json.dumps(d), flush=True)
            n += 1
print("searches", n, "errors", bad, "s", round(time.time() - t0, 1))
