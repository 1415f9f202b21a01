"""Prints SURVEY.md §6.1 (the C3 full sweep measured with the compiled
reference, one search() per pp job) from tests/golden/c3_full_ref.json."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
d = json.load(open(os.path.join(HERE, "..", "tests", "golden", "c3_full_ref.json")))
per = d["per_pp"]
walls = d["job_search_wall_s"]
cands = d["candidates_simulated"] + d["candidates_pruned"]
cpu = d["reference_cpu_seconds"]
print(f"Measured with the compiled, unmodified reference (`oracle/_ref`), one `search()` per pipeline-degree job "
      f"(`jobs = 1`, 6-8 jobs at a time on the build container's 8 cores, {d['cpu']}; "
      f"`tests/golden/gen_c3_full_ref.py` → `tests/golden/c3_full_ref.json`). Full mode has no cross-task "
      f"state, so the sweep is the concatenation of the per-pp searches.\n")
print(f"* Candidates: **{d['candidates_simulated']:,} simulated + {d['candidates_pruned']:,} pruned = {cands:,}**.")
print(f"* Best: {d['best_iteration_time_s']!r} s (bits {d['best_iteration_bits']}), the same plan as default mode.")
print(f"* Reference CPU time: **{cpu:,.0f} s = {cpu / 3600:.1f} CPU-hours** (sum of the jobs' `search()` walls); "
      f"{cands / cpu:,.0f} cand/s per core.")
big = sorted(walls.items(), key=lambda kv: -kv[1])[:6]
print("* Longest jobs: " + ", ".join(f"pp {k} {v / 60:.0f} min" for k, v in big) + ".\n")
print("| pp | simulated | pruned | log SHA-256 (first 12) |")
print("|---|---|---|---|")
for k in sorted(per, key=int):
    v = per[k]
    if int(k) % 8 == 0 or int(k) >= 84 or int(k) <= 2:
        print(f"| {k} | {v['simulated']:,} | {v['pruned']:,} | {v['sha256'][:12]} |")
print("\n(every pp in the JSON; the table shows a subset)")
