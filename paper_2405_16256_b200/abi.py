"""ctypes mirror of include/hetplan_b200.h plus conversion of the reference's
JSON documents (schema of /root/reference/proj/core/src/json_io.cpp:83-260)
into the flat hp_problem / hp_plan structs.

Defaults follow json_io.cpp exactly: group compute_efficiency 1.0 and
bwd_fwd_ratio 2.0 (:119-120), link latency 0 (:135), efficiency 0.85 for
gpu-direct / 0.76 for cpu-staged (:141-142), staging 16e9 for cpu-staged
(:144-146), planner defaults (:202-219).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Dict, List, NamedTuple, Tuple

HP_MAX_GROUPS = 16
HP_MAX_STAGES = 256

HP_OK, HP_BAD_CONFIG, HP_INFEASIBLE, HP_CUDA, HP_NCCL, HP_INTERNAL = range(6)
HP_GPIPE, HP_1F1B = 0, 1
HP_INTRA_NODE, HP_INTER_NODE, HP_INTER_GROUP = 0, 1, 2
HP_GPU_DIRECT, HP_CPU_STAGED = 0, 1
HP_REASON_COUNT = 4
HP_FLAG_TIME_KERNELS = 1
HP_FLAG_LOG = 2
REASONS = ("memory", "bound", "no_link", "no_assignment")


class hp_model(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_heads", C.c_int32), ("hidden_size", C.c_int64),
                ("seq_length", C.c_int64), ("vocab_size", C.c_int64), ("bytes_per_element", C.c_int32),
                ("_pad0", C.c_int32), ("activation_bytes_per_token_per_hidden", C.c_double),
                ("edge_layer_cost_multiplier", C.c_double)]


class hp_group(C.Structure):
    _fields_ = [("name", C.c_char_p), ("peak_tflops", C.c_double), ("memory_bytes", C.c_double),
                ("node_count", C.c_int32), ("devices_per_node", C.c_int32),
                ("compute_efficiency", C.c_double), ("bwd_fwd_ratio", C.c_double)]


class hp_link(C.Structure):
    _fields_ = [("scope", C.c_int32), ("path", C.c_int32), ("group_a", C.c_int32), ("group_b", C.c_int32),
                ("bandwidth_bits_per_s", C.c_double), ("latency_s", C.c_double), ("efficiency", C.c_double),
                ("staging_copy_bytes_per_s", C.c_double), ("group_a_name", C.c_char_p), ("group_b_name", C.c_char_p)]


class hp_cluster(C.Structure):
    _fields_ = [("n_groups", C.c_int32), ("n_links", C.c_int32), ("groups", C.POINTER(hp_group)),
                ("links", C.POINTER(hp_link))]


class hp_train(C.Structure):
    _fields_ = [("global_batch_size", C.c_int64), ("micro_batch_size", C.c_int64),
                ("optimizer_state_multiplier", C.c_double)]


class hp_planner(C.Structure):
    _fields_ = [("n_pipeline_degrees", C.c_int32), ("n_micro_batch_candidates", C.c_int32),
                ("pipeline_degrees", C.POINTER(C.c_int32)), ("micro_batch_candidates", C.POINTER(C.c_int64)),
                ("memory_headroom", C.c_double), ("exhaustive_split_limit", C.c_int64),
                ("stage_order_beam_width", C.c_int32), ("uniform_split_only", C.c_int32),
                ("allow_group_interleaving", C.c_int32), ("time_bound_pruning", C.c_int32),
                ("schedule", C.c_int32), ("_pad0", C.c_int32)]


class hp_problem(C.Structure):
    _fields_ = [("model", hp_model), ("cluster", hp_cluster), ("train", hp_train), ("planner", hp_planner)]


class hp_stage(C.Structure):
    _fields_ = [("layer_begin", C.c_int32), ("layer_end", C.c_int32), ("group", C.c_int32),
                ("nodes_used", C.c_int32), ("tp_degree", C.c_int32), ("dp_degree", C.c_int32)]


class hp_plan(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("schedule", C.c_int32), ("micro_batches_per_dp_replica", C.c_int64),
                ("micro_batch_size", C.c_int64), ("stages", hp_stage * HP_MAX_STAGES)]


class hp_search_opts(C.Structure):
    _fields_ = [("shard_index", C.c_int32), ("shard_count", C.c_int32), ("have_global_bound", C.c_int32),
                ("flags", C.c_int32), ("global_bound", C.c_double)]


class hp_result(C.Structure):
    _fields_ = [("candidates_simulated", C.c_int64), ("candidates_pruned", C.c_int64),
                ("reason_counts", C.c_int64 * HP_REASON_COUNT), ("leaves", C.c_int64), ("tasks", C.c_int64),
                ("has_best", C.c_int32), ("best_pp", C.c_int32), ("best_time_s", C.c_double),
                ("global_bound", C.c_double), ("device_ms", C.c_double), ("gpu_launches", C.c_int64),
                ("eval_launches", C.c_int64), ("eval_ms", C.c_double), ("eval_fp64_ops", C.c_double),
                ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double), ("host_ms", C.c_double),
                ("hill_iterations", C.c_int32), ("_pad1", C.c_int32), ("device_simulated", C.c_int64),
                ("device_aborted", C.c_int64), ("device_screened", C.c_int64), ("best_plan", hp_plan)]


class hp_trace_event(C.Structure):
    _fields_ = [("stage", C.c_int32), ("kind", C.c_int32), ("microbatch", C.c_int32), ("_pad", C.c_int32),
                ("start_s", C.c_double), ("end_s", C.c_double)]


class hp_stage_eval(C.Structure):
    _fields_ = [("fwd_s", C.c_double), ("bwd_s", C.c_double), ("send_fwd_s", C.c_double),
                ("send_bwd_s", C.c_double), ("dp_sync_s", C.c_double), ("busy_s", C.c_double),
                ("compute_end_s", C.c_double), ("bubble_ratio", C.c_double), ("peak_memory_bytes", C.c_double),
                ("peak_in_flight", C.c_int32), ("_pad", C.c_int32)]


class hp_plan_eval(C.Structure):
    _fields_ = [("iteration_time_s", C.c_double), ("pipeline_time_s", C.c_double),
                ("aggregate_bubble_ratio", C.c_double), ("micro_batches", C.c_int64), ("total_devices", C.c_int64),
                ("n_stages", C.c_int32), ("_pad", C.c_int32), ("n_trace", C.c_uint64)]


class hp_log_entry(C.Structure):
    _fields_ = [("candidate", C.c_uint64), ("reason", C.c_uint64), ("time_s", C.c_double),
                ("task", C.c_int32), ("leaf", C.c_int32)]


class SearchLogEntry(NamedTuple):
    """Reference SearchLogEntry (planner.hpp:95-99)."""
    candidate: str       # compact JSON descriptor
    time_s: float        # simulated time; -1.0 when pruned
    prune_reason: str    # "" when simulated


class ConfigError(ValueError):
    """Reference hetplan::ConfigError (errors.hpp:26-29)."""


class InfeasibleError(RuntimeError):
    """Reference hetplan::InfeasibleError (errors.hpp:39-44)."""

    def __init__(self, what, reasons=()):
        super().__init__(what)
        self.reasons = list(reasons)


class PlanError(RuntimeError):
    """Reference hetplan::PlanError (errors.hpp:31-37)."""

    def __init__(self, what, violations=()):
        super().__init__(what)
        self.violations = list(violations)


_SCOPES = {"intra-node": HP_INTRA_NODE, "inter-node-homogeneous": HP_INTER_NODE, "inter-group": HP_INTER_GROUP}
_PATHS = {"gpu-direct": HP_GPU_DIRECT, "cpu-staged": HP_CPU_STAGED}
_SCHED = {"gpipe": HP_GPIPE, "1f1b": HP_1F1B}


def _req(d, key, where):
    if key not in d:
        raise ConfigError(f"{where}: missing required field '{key}'")
    return d[key]


class Problem:
    """Owns an hp_problem and the arrays it points into."""

    def __init__(self, docs: Dict[str, dict]):
        m, c, t = docs["model"], docs["cluster"], docs["train"]
        p = docs.get("planner", {}) or {}
        self.struct = hp_problem()
        s = self.struct
        mm = s.model
        mm.num_layers = int(_req(m, "num_layers", "model"))
        mm.hidden_size = int(_req(m, "hidden_size", "model"))
        mm.seq_length = int(_req(m, "seq_length", "model"))
        mm.vocab_size = int(m.get("vocab_size", 0))
        mm.num_heads = int(_req(m, "num_heads", "model"))
        mm.bytes_per_element = int(m.get("bytes_per_element", 2))
        mm.activation_bytes_per_token_per_hidden = float(m.get("activation_bytes_per_token_per_hidden", 34.0))
        mm.edge_layer_cost_multiplier = float(m.get("edge_layer_cost_multiplier", 0.0))

        groups = _req(c, "groups", "cluster")
        links = _req(c, "links", "cluster")
        if len(groups) > HP_MAX_GROUPS:
            raise ConfigError(f"cluster: at most {HP_MAX_GROUPS} device groups supported")
        self.group_names: List[str] = []
        self._keep: List[bytes] = []  # name buffers the structs point into
        self._groups = (hp_group * max(1, len(groups)))()
        for i, g in enumerate(groups):
            name = str(_req(g, "name", "cluster.group"))
            self.group_names.append(name)
            G = self._groups[i]
            self._keep.append(name.encode())
            G.name = self._keep[-1]
            G.peak_tflops = float(_req(g, "peak_tflops", "cluster.group"))
            G.memory_bytes = float(_req(g, "memory_bytes", "cluster.group"))
            G.node_count = int(_req(g, "node_count", "cluster.group"))
            G.devices_per_node = int(_req(g, "devices_per_node", "cluster.group"))
            G.compute_efficiency = float(g.get("compute_efficiency", 1.0))
            G.bwd_fwd_ratio = float(g.get("bwd_fwd_ratio", 2.0))
        idx = {}
        for i, n in enumerate(self.group_names):
            idx.setdefault(n, i)
        self._links = (hp_link * max(1, len(links)))()
        for i, l in enumerate(links):
            ep = l.get("endpoints", l)
            kind = _req(ep, "kind", "cluster.link")
            if kind not in _SCOPES:
                raise ConfigError(f"cluster.link: unknown link kind '{kind}'")
            L = self._links[i]
            L.scope = _SCOPES[kind]
            # Unknown names map to -1 and are reported by the C-side
            # validation, which checks groups before links like
            # validate_spec (types.cpp:93-146). Duplicate names resolve to
            # the first declaration (find_group, types.cpp:26-31).
            if L.scope == HP_INTER_GROUP:
                a, b = _req(ep, "group_a", "cluster.link"), _req(ep, "group_b", "cluster.link")
                L.group_a, L.group_b = idx.get(a, -1), idx.get(b, -1)
                self._keep += [str(a).encode(), str(b).encode()]
                L.group_a_name, L.group_b_name = self._keep[-2], self._keep[-1]
            else:
                a = _req(ep, "group", "cluster.link")
                L.group_a, L.group_b = idx.get(a, -1), -1
                self._keep.append(str(a).encode())
                L.group_a_name = self._keep[-1]
            L.bandwidth_bits_per_s = float(_req(l, "bandwidth_bits_per_s", "cluster.link"))
            L.latency_s = float(l.get("latency_s", 0.0))
            pk = l.get("path_kind", "gpu-direct")
            if pk not in _PATHS:
                raise ConfigError(f"cluster.link: unknown path_kind '{pk}'")
            L.path = _PATHS[pk]
            L.efficiency = float(l.get("efficiency", 0.76 if L.path == HP_CPU_STAGED else 0.85))
            L.staging_copy_bytes_per_s = float(l.get("staging_copy_bytes_per_s",
                                                     16e9 if L.path == HP_CPU_STAGED else 0.0))
        s.cluster.n_groups = len(groups)
        s.cluster.n_links = len(links)
        s.cluster.groups = self._groups
        s.cluster.links = self._links

        s.train.global_batch_size = int(_req(t, "global_batch_size", "train"))
        s.train.micro_batch_size = int(_req(t, "micro_batch_size", "train"))
        s.train.optimizer_state_multiplier = float(t.get("optimizer_state_multiplier", 8.0))

        pps = [int(x) for x in p.get("pipeline_degrees", [])]
        mbs = [int(x) for x in p.get("micro_batch_candidates", [])]
        self._pps = (C.c_int32 * max(1, len(pps)))(*pps)
        self._mbs = (C.c_int64 * max(1, len(mbs)))(*mbs)
        pl = s.planner
        pl.n_pipeline_degrees = len(pps)
        pl.pipeline_degrees = self._pps
        pl.n_micro_batch_candidates = len(mbs)
        pl.micro_batch_candidates = self._mbs
        pl.uniform_split_only = int(bool(p.get("uniform_split_only", False)))
        pl.memory_headroom = float(p.get("memory_headroom", 0.9))
        pl.stage_order_beam_width = int(p.get("stage_order_beam_width", 24))
        pl.exhaustive_split_limit = int(p.get("exhaustive_split_limit", 2000))
        pl.allow_group_interleaving = int(bool(p.get("allow_group_interleaving", False)))
        pl.time_bound_pruning = int(bool(p.get("time_bound_pruning", True)))
        sched = p.get("schedule", "1f1b")
        if sched not in _SCHED:
            raise ConfigError(f"planner: unknown schedule '{sched}'")
        pl.schedule = _SCHED[sched]

    def ptr(self):
        return C.byref(self.struct)

    # ---- plan conversion (json_io.cpp:233-278) ----
    def plan_from_doc(self, d: dict) -> hp_plan:
        p = hp_plan()
        p.schedule = _SCHED[d["schedule"]]
        p.micro_batches_per_dp_replica = int(d["micro_batches_per_dp_replica"])
        p.micro_batch_size = int(d.get("micro_batch_size", 0))
        st = d["stages"]
        if len(st) > HP_MAX_STAGES:
            raise ConfigError("plan: too many stages")
        p.n_stages = len(st)
        gi = {n: i for i, n in enumerate(self.group_names)}
        for i, s in enumerate(st):
            S = p.stages[i]
            S.layer_begin, S.layer_end = s["layer_range"]
            S.group = gi[s["group"]]
            S.nodes_used, S.tp_degree, S.dp_degree = s["nodes_used"], s["tp_degree"], s["dp_degree"]
        return p

    def plan_to_doc(self, p: hp_plan) -> dict:
        return {"schema_version": 1, "schedule": "gpipe" if p.schedule == HP_GPIPE else "1f1b",
                "micro_batches_per_dp_replica": int(p.micro_batches_per_dp_replica),
                "micro_batch_size": int(p.micro_batch_size),
                "stages": [{"layer_range": [p.stages[i].layer_begin, p.stages[i].layer_end],
                            "group": self.group_names[p.stages[i].group],
                            "nodes_used": p.stages[i].nodes_used, "tp_degree": p.stages[i].tp_degree,
                            "dp_degree": p.stages[i].dp_degree} for i in range(p.n_stages)]}


def encode_plan(group_names, p: hp_plan) -> str:
    """encode_plan (planner.cpp:192-200)."""
    s = ("gpipe" if p.schedule == HP_GPIPE else "1f1b") + f"|{p.micro_batches_per_dp_replica}|{p.micro_batch_size}"
    for i in range(p.n_stages):
        st = p.stages[i]
        s += f"|{group_names[st.group]}:{st.layer_begin}-{st.layer_end}:{st.nodes_used}:{st.tp_degree}:{st.dp_degree}"
    return s


def better_key(group_names, time_s: float, pp: int, p: hp_plan) -> Tuple[float, int, bytes]:
    """Sort key equal to better_than (planner.cpp:178-183); std::string
    operator< compares bytes as unsigned char... as char — ASCII here."""
    return (time_s, pp, encode_plan(group_names, p).encode())


INF = math.inf
