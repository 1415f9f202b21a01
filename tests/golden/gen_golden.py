"""Generates the golden fixtures in tests/golden/ by running the compiled,
unmodified reference planner (oracle/_ref, built from /root/reference by
oracle/Makefile). Run in the build container:

    make -C oracle ref && python tests/golden/gen_golden.py

Fixtures pin: search() outcomes (plan, iteration-time bits, candidate counts)
on the shipped sample (C0), C1 and C2u in both pruning modes and on seeded
random small instances covering both schedules, exhaustive and hill-climb
split search, group interleaving, uniform-only search, infeasible inputs and
cpu-staged links; split_layers (planner.cpp:42-84) and simulate()
(sim.cpp:63-195) on seeded random inputs.
"""
from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2405_16256_b200 import configs  # noqa: E402
from tests.instances import random_instance  # noqa: E402


def search_case(name, cfg):
    r = ref.search(cfg, jobs=4)
    case = {"name": name, "docs": cfg, "status": r["status"]}
    if r["status"] == 0:
        case.update({"plan": r["plan"], "iteration_bits": r["eval"]["iteration_bits"],
                     "iteration_time_s": r["eval"]["iteration_time_s"],
                     "candidates_simulated": r["candidates_simulated"],
                     "candidates_pruned": r["candidates_pruned"]})
    else:
        case["error"] = r.get("error")
        case["reasons"] = r.get("reasons", [])[:5]
    return case


def main():
    cases = []
    for n in ["C0", "C1", "C2u"]:
        for full in (True, False):
            cases.append(search_case(f"{n}-{'full' if full else 'default'}", configs.config(n, full=full)))
    cases.append(search_case("C2-default", configs.config("C2", full=False)))
    cases.append(search_case("C3pp12-full", configs.with_pp(configs.config("C3", full=True), [12])))
    rng = random.Random(20261018)
    for k in range(160):
        cfg = random_instance(rng, k)
        cases.append(search_case(f"rand{k:03d}", cfg))
    with open(os.path.join(HERE, "search_cases.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))

    # split_layers fixtures (test_planner.cpp:114-143 style, seeded)
    rng = random.Random(2026)
    splits = [{"total": 80, "w": [1.0] * 10}, {"total": 10, "w": [2.0, 1.0, 1.0]}, {"total": 7, "w": [1.0, 1.0]},
              {"total": 3, "w": [100.0, 1.0, 1.0]}]
    for total in range(1, 31):
        for stages in range(1, min(6, total) + 1):
            for _ in range(3):
                splits.append({"total": total, "w": [rng.uniform(0.05, 10.0) for _ in range(stages)]})
    for s in splits:
        s["out"] = ref.split_layers(s["total"], s["w"])
    with open(os.path.join(HERE, "split_layers.json"), "w") as f:
        json.dump(splits, f, separators=(",", ":"))

    # simulate fixtures (test_sim.cpp random_times style, seeded)
    rng = random.Random(42)
    sims = []
    for trial in range(120):
        P = 1 + rng.randrange(12)
        M = 1 + rng.randrange(40)
        gpipe = trial % 3 == 0
        times = []
        for _ in range(P):
            f = rng.uniform(0.0, 2.0)
            times.append([f, f + rng.uniform(0.0, 2.0), 0.5 * rng.uniform(0.0, 2.0), 0.5 * rng.uniform(0.0, 2.0)])
        it, ce = ref.simulate(times, M, gpipe)
        sims.append({"P": P, "M": M, "gpipe": gpipe, "times": times, "iteration": it, "compute_end": ce,
                     "iteration_bits": float(it).hex()})
    with open(os.path.join(HERE, "simulate.json"), "w") as f:
        json.dump(sims, f, separators=(",", ":"))
    print(f"{len(cases)} search cases, {len(splits)} split_layers cases, {len(sims)} simulate cases")


if __name__ == "__main__":
    main()
