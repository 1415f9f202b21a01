"""Generates tests/golden/gpipe_scale.json: GPipe (sim.cpp:46-50) at scale,
pinned by the compiled, unmodified reference (oracle/_ref) — the generic
counter-driven evaluator's regime (hp_kernels.cu eval_item_generic), which
the reference's own tests only cover at small P*M.

* C3 (Llama-140B, 768 devices) with schedule gpipe, memory unbounded (GPipe
  retains all M activations), full mode, pipeline degree 64, micro-batch 1:
  P*M up to 98,304 per candidate.

    python tests/golden/gen_gpipe_scale.py [--jobs 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from paper_2405_16256_b200 import configs  # noqa: E402


def docs():
    d = configs.with_pp(configs.config("C3", full=True), [64])
    d["planner"]["schedule"] = "gpipe"
    d["planner"]["micro_batch_candidates"] = [1]
    for g in d["cluster"]["groups"]:
        g["memory_bytes"] = 1e18
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=4)
    a = ap.parse_args()
    d = docs()
    r = ref.search(d, jobs=a.jobs)
    rec = {"name": "C3-gpipe-pp64-B1", "docs": d, "status": r["status"], "wall_s": r.get("wall_s"), "jobs": a.jobs,
           "iteration_bits": r["eval"]["iteration_bits"], "plan": r["plan"],
           "candidates_simulated": r["candidates_simulated"], "candidates_pruned": r["candidates_pruned"]}
    with open(os.path.join(HERE, "gpipe_scale.json"), "w") as f:
        json.dump(rec, f, indent=0)
    print(rec["status"], rec["candidates_simulated"], rec["candidates_pruned"], rec["wall_s"])


if __name__ == "__main__":
    main()
