"""Synthetic planner inputs C0..C5, as the reference's own
JSON documents (model / cluster / train / planner, schema of
/root/reference/proj/core/src/json_io.cpp:83-219).

Shared values come from the reference's shipped sample
(proj/configs/cluster_12n_1to5.json:1-36, model_llama2_70b.json:1-10) and the
paper (PAPER.md:391 for Llama-140B, PAPER.md:582 for homogeneous MFUs).
All inputs are deterministic; nothing here is random.
"""
from __future__ import annotations

import copy
from typing import Dict

LLAMA = {
    "7b": {"num_layers": 32, "hidden_size": 4096, "seq_length": 4096, "num_heads": 32},
    "70b": {"num_layers": 80, "hidden_size": 8192, "seq_length": 4096, "num_heads": 64},
    "140b": {"num_layers": 160, "hidden_size": 8192, "seq_length": 4096, "num_heads": 64},
}

# cluster_12n_1to5.json:3-20 plus synthetic peaks from SURVEY.md §8d (C4/C5).
GROUP_PRESETS = {
    "amd": {"peak_tflops": 383.0, "compute_efficiency": 0.245, "memory_bytes": 64e9},
    "gpu_a": {"peak_tflops": 147.0, "compute_efficiency": 0.327, "memory_bytes": 64e9},
}
C4_TYPES = {
    "nvidia": {"peak_tflops": 312.0, "compute_efficiency": 0.564, "memory_bytes": 80e9},
    "gpu_a": {"peak_tflops": 147.0, "compute_efficiency": 0.453, "memory_bytes": 64e9},
    "amd": {"peak_tflops": 383.0, "compute_efficiency": 0.389, "memory_bytes": 64e9},
    "gpu_b": {"peak_tflops": 256.0, "compute_efficiency": 0.288, "memory_bytes": 64e9},
}


def model_doc(size: str) -> dict:
    d = dict(LLAMA[size])
    d.update({"vocab_size": 32000, "bytes_per_element": 2,
              "activation_bytes_per_token_per_hidden": 34, "edge_layer_cost_multiplier": 0})
    return d


def group(name: str, preset: dict, nodes: int, dpn: int, **over) -> dict:
    g = {"name": name, "node_count": nodes, "devices_per_node": dpn, "bwd_fwd_ratio": 2.0}
    g.update(preset)
    g.update(over)
    return g


def links_for(groups) -> list:
    """Intra 4.8e12 b/s eff .85, inter-node 200e9 eff .85, every group pair
    cpu-staged 25e9 eff .76 staging 16e9 latency 20us (cluster_12n_1to5.json:22-35)."""
    links = []
    for g in groups:
        links.append({"endpoints": {"kind": "intra-node", "group": g["name"]},
                      "bandwidth_bits_per_s": 4.8e12, "efficiency": 0.85})
        links.append({"endpoints": {"kind": "inter-node-homogeneous", "group": g["name"]},
                      "bandwidth_bits_per_s": 200e9, "efficiency": 0.85})
    for a in range(len(groups)):
        for b in range(a + 1, len(groups)):
            links.append({"endpoints": {"kind": "inter-group", "group_a": groups[a]["name"],
                                        "group_b": groups[b]["name"]},
                          "bandwidth_bits_per_s": 25e9, "efficiency": 0.76,
                          "path_kind": "cpu-staged", "staging_copy_bytes_per_s": 16e9,
                          "latency_s": 20e-6})
    return links


def cluster_doc(groups) -> dict:
    return {"groups": groups, "links": links_for(groups)}


def planner_doc(**kw) -> dict:
    p = {"memory_headroom": 0.9, "stage_order_beam_width": 24,
         "exhaustive_split_limit": 2000, "schedule": "1f1b"}
    p.update(kw)
    return p


def config(name: str, full: bool = True) -> Dict[str, dict]:
    """Returns {"model","cluster","train","planner"} for C0..C5.

    ``full`` selects the reference's "full strategy sweep" mode
    (time_bound_pruning=false, planner.hpp:44-47); False keeps the CLI
    default (pruning on, json_io.cpp:215)."""
    prune = {"time_bound_pruning": not full}
    if name == "C0":  # shipped sample, no profiles (proj/configs/*.json)
        groups = [group("amd", GROUP_PRESETS["amd"], 2, 8), group("gpu_a", GROUP_PRESETS["gpu_a"], 10, 8)]
        return {"model": model_doc("70b"), "cluster": cluster_doc(groups),
                "train": {"global_batch_size": 256, "micro_batch_size": 1, "optimizer_state_multiplier": 8.0},
                "planner": planner_doc(pipeline_degrees=[6, 12, 24], micro_batch_candidates=[1, 2], **prune)}
    if name == "C1":  # Llama-7B on 8+8 single-device nodes
        groups = [group("amd", GROUP_PRESETS["amd"], 8, 1), group("gpu_a", GROUP_PRESETS["gpu_a"], 8, 1)]
        return {"model": model_doc("7b"), "cluster": cluster_doc(groups),
                "train": {"global_batch_size": 64, "micro_batch_size": 1, "optimizer_state_multiplier": 8.0},
                "planner": planner_doc(micro_batch_candidates=[1, 2, 4], **prune)}
    if name in ("C2", "C2u"):  # Llama-70B on 256 devices, uniform vs non-uniform
        groups = [group("amd", GROUP_PRESETS["amd"], 6, 8), group("gpu_a", GROUP_PRESETS["gpu_a"], 26, 8)]
        return {"model": model_doc("70b"), "cluster": cluster_doc(groups),
                "train": {"global_batch_size": 512, "micro_batch_size": 1, "optimizer_state_multiplier": 8.0},
                "planner": planner_doc(micro_batch_candidates=[1, 2], uniform_split_only=(name == "C2u"), **prune)}
    if name == "C3":  # Llama-140B on 768 devices (128 AMD + 640 gpu_a), paper headline
        groups = [group("amd", GROUP_PRESETS["amd"], 16, 8), group("gpu_a", GROUP_PRESETS["gpu_a"], 80, 8)]
        return {"model": model_doc("140b"), "cluster": cluster_doc(groups),
                "train": {"global_batch_size": 1536, "micro_batch_size": 1, "optimizer_state_multiplier": 8.0},
                "planner": planner_doc(micro_batch_candidates=[1, 2], **prune)}
    if name.startswith("C4"):  # C4:<a>+<b>, Llama-70B, 32+32 nodes x 8
        a, b = name.split(":")[1].split("+")
        groups = [group(a, C4_TYPES[a], 32, 8), group(b, C4_TYPES[b], 32, 8)]
        return {"model": model_doc("70b"), "cluster": cluster_doc(groups),
                "train": {"global_batch_size": 1024, "micro_batch_size": 1, "optimizer_state_multiplier": 8.0},
                "planner": planner_doc(micro_batch_candidates=[1, 2], **prune)}
    if name == "C5":  # stress: 3 types, 160 layers, exhaustive splits at pp 3/4
        big = {"memory_bytes": 192e9}
        groups = [group("amd", GROUP_PRESETS["amd"], 8, 8, **big),
                  group("gpu_a", GROUP_PRESETS["gpu_a"], 16, 8, **big),
                  group("gpu_c", {"peak_tflops": 200.0, "compute_efficiency": 0.353}, 8, 8, **big)]
        return {"model": model_doc("140b"), "cluster": cluster_doc(groups),
                "train": {"global_batch_size": 1024, "micro_batch_size": 1, "optimizer_state_multiplier": 8.0},
                "planner": planner_doc(pipeline_degrees=[3, 4], micro_batch_candidates=[1, 2, 4, 8],
                                       exhaustive_split_limit=1000000, time_bound_pruning=False)}
    raise KeyError(name)


C4_PAIRS = ["nvidia+gpu_a", "nvidia+amd", "nvidia+gpu_b", "gpu_a+amd", "gpu_a+gpu_b", "amd+gpu_b"]


def with_pp(cfg: Dict[str, dict], pps) -> Dict[str, dict]:
    c = copy.deepcopy(cfg)
    c["planner"]["pipeline_degrees"] = list(pps)
    return c
