"""Seeded random planner instances (small enough for the CPU oracle), in the
reference's JSON document schema. Modelled on the reference tests' builders
(tests/test_util.hpp:26-136: two_group_cluster, one_group_cluster,
tiny_model, train_config) but drawn over all planner options."""
from __future__ import annotations

import random

NAMES = ["fast", "slow", "gpu", "amd", "a", "bb", "gpu_x", "n1"]


def random_instance(rng: random.Random, k: int = 0) -> dict:
    n_groups = rng.choice([1, 2, 2, 2, 3])
    names = rng.sample(NAMES, n_groups)
    groups = []
    for nm in names:
        groups.append({
            "name": nm,
            "peak_tflops": round(rng.uniform(50, 400), 3),
            "memory_bytes": rng.choice([1e18, 1e18, 64e9, 16e9, 4e9, 1e9]),
            "node_count": rng.randint(1, 4),
            "devices_per_node": rng.choice([1, 1, 2, 4, 8]),
            "compute_efficiency": round(rng.uniform(0.2, 1.0), 4),
            "bwd_fwd_ratio": round(rng.uniform(1.0, 3.0), 3),
        })
    links = []
    for nm in names:
        links.append({"endpoints": {"kind": "intra-node", "group": nm},
                      "bandwidth_bits_per_s": rng.choice([1e12, 4.8e12, 2e11]),
                      "efficiency": rng.choice([0.85, 1.0, 0.6]),
                      "latency_s": rng.choice([0.0, 0.0, 1e-6])})
        links.append({"endpoints": {"kind": "inter-node-homogeneous", "group": nm},
                      "bandwidth_bits_per_s": rng.choice([2e11, 1e11, 4e11]),
                      "efficiency": rng.choice([0.85, 0.9]),
                      "latency_s": rng.choice([0.0, 5e-6])})
    for a in range(n_groups):
        for b in range(a + 1, n_groups):
            if rng.random() < 0.85:
                staged = rng.random() < 0.5
                l = {"endpoints": {"kind": "inter-group", "group_a": names[a], "group_b": names[b]},
                     "bandwidth_bits_per_s": rng.choice([25e9, 5e9, 1e11]),
                     "latency_s": rng.choice([0.0, 2e-5])}
                if staged:
                    l["path_kind"] = "cpu-staged"
                    l["staging_copy_bytes_per_s"] = rng.choice([16e9, 8e9])
                else:
                    l["efficiency"] = 0.85
                links.append(l)
    H = rng.choice([64, 128, 256, 512, 1024, 4096])
    model = {"num_layers": rng.randint(2, 24), "hidden_size": H, "seq_length": rng.choice([64, 128, 512, 2048]),
             "vocab_size": 1000, "num_heads": rng.choice([1, 2, 4, 8]), "bytes_per_element": rng.choice([2, 2, 4]),
             "activation_bytes_per_token_per_hidden": 34, "edge_layer_cost_multiplier": rng.choice([0, 0, 0.5])}
    G = rng.choice([4, 8, 12, 16, 32, 64])
    train = {"global_batch_size": G, "micro_batch_size": rng.choice([1, 1, 2]), "optimizer_state_multiplier": 8.0}
    total_nodes = sum(g["node_count"] for g in groups)
    cap = min(model["num_layers"], total_nodes, 8)
    planner = {"memory_headroom": rng.choice([1.0, 0.9, 0.5]),
               "stage_order_beam_width": rng.choice([0, 1, 2, 24]),
               "exhaustive_split_limit": rng.choice([0, 10, 200, 2000]),
               "allow_group_interleaving": rng.random() < 0.2,
               "time_bound_pruning": rng.random() < 0.5,
               "schedule": "gpipe" if rng.random() < 0.25 else "1f1b",
               "uniform_split_only": rng.random() < 0.08}
    if rng.random() < 0.7:
        planner["pipeline_degrees"] = sorted(rng.sample(range(1, cap + 1), rng.randint(1, cap)))
    if rng.random() < 0.6:
        planner["micro_batch_candidates"] = sorted(rng.sample([1, 2, 4], rng.randint(1, 3)))
    return {"model": model, "cluster": {"groups": groups, "links": links}, "train": train, "planner": planner}
