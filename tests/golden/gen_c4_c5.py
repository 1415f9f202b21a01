"""Generates tests/golden/c4_c5_cases.json: golden search outcomes of the
compiled, UNMODIFIED reference (oracle/_ref) on SURVEY.md §8d's C4 and C5.

* C4 (Llama-70B, 512 devices, all six accelerator pairs): default mode
  (time_bound_pruning = true, the CLI default, json_io.cpp:215) over the
  whole pp range, with the search-log digest; full mode (pruning off) on the
  pipeline degrees {2, 4, 6, 8, 10, 12} (the reference needs ~6 min at pp 32
  alone, so the full pp range is hours per pair).
* C5 (160 layers, 3 device types, exhaustive splits up to 1e6 per leaf):
  pp 3 with micro-batch sizes 4, 2 and 1 — every composition of every leaf
  enumerated (planner.cpp:454-459); at micro-batch 8 every candidate is
  memory-pruned (InfeasibleError), so that slice would pin nothing. pp 4 (657,359 compositions per
  leaf, ~1.8e9 candidates per micro-batch size) is beyond the reference's
  reach on a CPU and is pinned on the GPU by the C restatement and properties.

Records use the search_cases.json format (docs, status, iteration_bits,
counts, plan) plus wall seconds, so tests/test_gpu_parity.py's check_case
applies unchanged.

    python tests/golden/gen_c4_c5.py [--jobs 2]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2405_16256_b200 import configs  # noqa: E402

C4_FULL_PP = [2, 4, 6, 8, 10, 12]
OUT = os.path.join(HERE, "c4_c5_cases.json")


def digest(log) -> str:
    h = hashlib.sha256()
    for e in log:
        h.update(f"{e['candidate']}\t{e['time_bits']}\t{e['reason']}\n".encode())
    return h.hexdigest()


def cases():
    for pair in configs.C4_PAIRS:
        yield f"C4:{pair}:default", configs.config("C4:" + pair, full=False), True
        yield f"C4:{pair}:full:pp{C4_FULL_PP}", configs.with_pp(configs.config("C4:" + pair, full=True), C4_FULL_PP), False
    for B in (4, 2, 1):
        d = configs.with_pp(configs.config("C5"), [3])
        d["planner"]["micro_batch_candidates"] = [B]
        yield f"C5:pp3:B{B}", d, False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=2)
    a = ap.parse_args()
    done = {c["name"]: c for c in json.load(open(OUT))} if os.path.exists(OUT) else {}
    for name, docs, want_log in cases():
        if name in done:
            continue
        r = ref.search(docs, jobs=a.jobs, want_log=want_log)
        rec = {"name": name, "docs": docs, "status": r["status"], "wall_s": r.get("wall_s"), "jobs": a.jobs}
        if r["status"] == 0:
            rec.update({"iteration_bits": r["eval"]["iteration_bits"], "plan": r["plan"],
                        "candidates_simulated": r["candidates_simulated"],
                        "candidates_pruned": r["candidates_pruned"]})
            if want_log:
                rec["log"] = {"n": len(r["log"]), "sha256": digest(r["log"])}
        else:
            rec["error"] = r.get("error")
        done[name] = rec
        print(name, rec["status"], rec.get("candidates_simulated"), rec.get("candidates_pruned"), rec["wall_s"],
              flush=True)
        with open(OUT + ".tmp", "w") as f:
            json.dump(list(done.values()), f, indent=0)
        os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main()
