"""Generates tests/golden/climb_cases.json: seeded random instances where the
full-sweep hill climb does the work (more layers and stages than
tests/instances.py, many microbatches, exhaustive enumeration off or
small) and groups are joined by slow, often cpu-staged links — the inputs
on which the GPU's neighbour screen (per-stage and pair-circuit bounds,
hp_search_core.cuh) skips most neighbours. Outcomes come from the compiled,
unmodified reference planner (oracle/_ref). Run in the build container:

    make -C oracle ref && python tests/golden/gen_climb_cases.py
"""
from __future__ import annotations

import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

NAMES = ["fast", "slow", "gpu", "amd", "npu"]


def climb_instance(rng: random.Random) -> dict:
    n_groups = rng.choice([2, 2, 3])
    names = rng.sample(NAMES, n_groups)
    groups = [{"name": nm, "peak_tflops": round(rng.uniform(80, 400), 3),
               "memory_bytes": rng.choice([1e18, 1e18, 80e9]), "node_count": rng.randint(2, 8),
               "devices_per_node": rng.choice([1, 2, 8]), "compute_efficiency": round(rng.uniform(0.3, 0.9), 4),
               "bwd_fwd_ratio": round(rng.uniform(1.5, 2.5), 3)} for nm in names]
    links = []
    for nm in names:
        links.append({"endpoints": {"kind": "intra-node", "group": nm}, "bandwidth_bits_per_s": 4.8e12,
                      "efficiency": 0.85, "latency_s": 0.0})
        links.append({"endpoints": {"kind": "inter-node-homogeneous", "group": nm},
                      "bandwidth_bits_per_s": rng.choice([2e11, 4e11]), "efficiency": 0.9,
                      "latency_s": rng.choice([0.0, 5e-6])})
    for a in range(n_groups):
        for b in range(a + 1, n_groups):
            l = {"endpoints": {"kind": "inter-group", "group_a": names[a], "group_b": names[b]},
                 "bandwidth_bits_per_s": rng.choice([5e9, 25e9, 1e11]), "latency_s": rng.choice([0.0, 2e-5])}
            if rng.random() < 0.5:
                l["path_kind"] = "cpu-staged"
                l["staging_copy_bytes_per_s"] = rng.choice([8e9, 16e9])
            else:
                l["efficiency"] = 0.85
            links.append(l)
    L = rng.randint(24, 64)
    model = {"num_layers": L, "hidden_size": rng.choice([1024, 2048, 4096]), "seq_length": rng.choice([512, 2048]),
             "vocab_size": 32000, "num_heads": 16, "bytes_per_element": 2,
             "activation_bytes_per_token_per_hidden": 34, "edge_layer_cost_multiplier": rng.choice([0, 0.5])}
    train = {"global_batch_size": rng.choice([64, 128, 256, 512]), "micro_batch_size": 1,
             "optimizer_state_multiplier": 8.0}
    total_nodes = sum(g["node_count"] for g in groups)
    cap = min(L, total_nodes, 24)
    lo = max(2, cap // 3)
    planner = {"memory_headroom": 0.9, "stage_order_beam_width": rng.choice([1, 2, 4]),
               "exhaustive_split_limit": rng.choice([0, 0, 10]), "allow_group_interleaving": False,
               "time_bound_pruning": False, "schedule": "gpipe" if rng.random() < 0.2 else "1f1b",
               "pipeline_degrees": sorted(rng.sample(range(lo, cap + 1), min(3, cap - lo + 1))),
               "micro_batch_candidates": rng.choice([[1], [1, 2]])}
    return {"model": model, "cluster": {"groups": groups, "links": links}, "train": train, "planner": planner}


def main():
    rng = random.Random(20261019)
    jobs = int(os.environ.get("JOBS", os.cpu_count() or 4))
    cases = []
    for k in range(int(os.environ.get("N_CASES", 60))):
        cfg = climb_instance(rng)
        t0 = time.time()
        r = ref.search(cfg, jobs=jobs)
        case = {"name": f"climb{k:02d}", "docs": cfg, "status": r["status"], "ref_s": round(time.time() - t0, 2)}
        if r["status"] == 0:
            case.update({"plan": r["plan"], "iteration_bits": r["eval"]["iteration_bits"],
                         "iteration_time_s": r["eval"]["iteration_time_s"],
                         "candidates_simulated": r["candidates_simulated"],
                         "candidates_pruned": r["candidates_pruned"]})
        else:
            case["error"] = r.get("error")
        print(case["name"], case["status"], case.get("candidates_simulated"), case["ref_s"], flush=True)
        cases.append(case)
    with open(os.path.join(HERE, "climb_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/gen_climb_cases.py (oracle/_ref, the compiled reference)",
                   "cases": cases}, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
