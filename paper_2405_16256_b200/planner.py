"""Host-side mirror of the reference planner interface for the hot path.

    search(docs, jobs=1, log=False) -> SearchOutcome   (planner.hpp:115-116)
    evaluate_plans(docs, plans) -> [iteration_time_s]  (evaluate.hpp:56-58, batched)
    evaluate_plan(docs, plan, trace) -> PlanEvaluation  (evaluate.hpp:56-58, record_trace)

`docs` are the reference's own JSON documents {"model","cluster","train",
"planner"} (json_io.cpp:83-219). Errors raise the reference's exception kinds
(ConfigError / InfeasibleError, errors.hpp:26-44). The work runs in the
sm_100a CUDA library through the C ABI of include/hetplan_b200.h; there is no
CPU fallback. Multi-GPU: search_sharded() runs one shard per rank and reduces
the per-rank best records with one NCCL all-gather (torch.distributed).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import abi
from ._lib import lib


@dataclass
class SearchOutcome:
    plan: dict
    iteration_time_s: float
    candidates_simulated: int
    candidates_pruned: int
    reason_counts: Dict[str, int] = field(default_factory=dict)
    device_ms: float = 0.0
    gpu_launches: int = 0
    leaves: int = 0
    tasks: int = 0
    global_bound: float = math.inf
    raw: Optional[abi.hp_result] = None
    log: List[abi.SearchLogEntry] = field(default_factory=list)  # SearchOutcome::log (when requested)


class Engine:
    """One hp_ctx bound to one CUDA device (reused across searches)."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        self._ctx = C.c_void_p()
        st = self._lib.hp_create(C.byref(self._ctx), device)
        if st != abi.HP_OK:
            raise RuntimeError(f"hp_create(device={device}) failed with status {st}")
        self.device = device

    def close(self):
        if self._ctx:
            self._lib.hp_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, st: int, what: str):
        msg = (self._lib.hp_last_error(self._ctx) or b"").decode()
        if st == abi.HP_BAD_CONFIG:
            raise abi.ConfigError(msg)
        if st == abi.HP_INFEASIBLE:
            raise abi.InfeasibleError(msg or "no feasible plan found")
        raise RuntimeError(f"{what} failed (status {st}): {msg}")

    def search_shard(self, problem: abi.Problem, shard_index: int = 0, shard_count: int = 1,
                     global_bound: Optional[float] = None, flags: int = 0) -> abi.hp_result:
        opts = abi.hp_search_opts(shard_index, shard_count, int(global_bound is not None), flags,
                                  global_bound if global_bound is not None else 0.0)
        res = abi.hp_result()
        st = self._lib.hp_search(self._ctx, problem.ptr(), C.byref(opts), C.byref(res))
        if st != abi.HP_OK:
            self._raise(st, "hp_search")
        return res

    def search_log(self) -> List[Tuple[int, int, abi.SearchLogEntry]]:
        """The log of the last search_shard(flags=HP_FLAG_LOG): (task, leaf,
        entry) in the reference's order for this shard."""
        n = C.c_uint64()
        nb = C.c_uint64()
        st = self._lib.hp_search_log(self._ctx, None, 0, None, 0, C.byref(n), C.byref(nb))
        if st != abi.HP_OK:
            self._raise(st, "hp_search_log")
        ents = (abi.hp_log_entry * max(1, n.value))()
        text = C.create_string_buffer(max(1, nb.value))
        st = self._lib.hp_search_log(self._ctx, ents, n.value, text, nb.value, C.byref(n), C.byref(nb))
        if st != abi.HP_OK:
            self._raise(st, "hp_search_log")
        raw = text.raw
        out = []
        for k in range(n.value):
            e = ents[k]
            c0 = e.candidate
            r0 = e.reason
            cand = raw[c0:raw.index(b"\0", c0)].decode()
            reason = raw[r0:raw.index(b"\0", r0)].decode()
            out.append((e.task, e.leaf, abi.SearchLogEntry(cand, e.time_s, reason)))
        return out

    def probe_shard(self, problem: abi.Problem, shard_index: int = 0, shard_count: int = 1) -> float:
        opts = abi.hp_search_opts(shard_index, shard_count, 0, 0, 0.0)
        b = C.c_double()
        st = self._lib.hp_probe(self._ctx, problem.ptr(), C.byref(opts), C.byref(b))
        if st != abi.HP_OK:
            self._raise(st, "hp_probe")
        return b.value

    def evaluate_plans(self, problem: abi.Problem, plans: List[abi.hp_plan]) -> List[float]:
        n = len(plans)
        arr = (abi.hp_plan * max(1, n))(*plans)
        out = (C.c_double * max(1, n))()
        st = self._lib.hp_evaluate_plans(self._ctx, problem.ptr(), arr, n, out)
        if st != abi.HP_OK:
            self._raise(st, "hp_evaluate_plans")
        return list(out)[:n]


    def evaluate_plan_full(self, problem: abi.Problem, plan: abi.hp_plan, trace: bool = True) -> "PlanEvaluation":
        ev = abi.hp_plan_eval()
        st = (abi.hp_stage_eval * max(1, plan.n_stages))()
        n_tr = 4 * plan.n_stages * plan.micro_batches_per_dp_replica - 2 * plan.micro_batches_per_dp_replica
        tr = (abi.hp_trace_event * max(1, n_tr))() if trace else None
        rc = self._lib.hp_evaluate_plan_full(self._ctx, problem.ptr(), C.byref(plan), C.byref(ev), st, tr,
                                             n_tr if trace else 0)
        if rc != abi.HP_OK:
            self._raise(rc, "hp_evaluate_plan_full")
        return PlanEvaluation(ev, [st[i] for i in range(plan.n_stages)],
                              [tr[i] for i in range(ev.n_trace)] if trace else [])


@dataclass
class PlanEvaluation:
    """PlanEvaluation of evaluate.hpp:38-44 (with SimResult, sim.hpp:44-53):
    scalars in `eval`, per-stage vectors in `stages`, the sorted trace."""
    eval: abi.hp_plan_eval
    stages: List[abi.hp_stage_eval]
    trace: List[abi.hp_trace_event]


class MultiEngine:
    """hp_multi: one context per listed GPU in this process, NCCL between
    them (include/hetplan_b200.h hp_search_multi)."""

    def __init__(self, devices: List[int]):
        self._lib = lib()
        self._m = C.c_void_p()
        arr = (C.c_int32 * len(devices))(*devices)
        st = self._lib.hp_multi_create(C.byref(self._m), arr, len(devices))
        if st != abi.HP_OK:
            msg = (self._lib.hp_multi_last_error(self._m) or b"").decode()
            self.close()
            raise RuntimeError(f"hp_multi_create({devices}) failed with status {st}: {msg}")
        self.devices = list(devices)

    def close(self):
        if self._m:
            self._lib.hp_multi_destroy(self._m)
            self._m = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, problem: abi.Problem, flags: int = 0) -> Tuple[abi.hp_result, List[abi.hp_result]]:
        red = abi.hp_result()
        per = (abi.hp_result * len(self.devices))()
        st = self._lib.hp_search_multi(self._m, problem.ptr(), flags, C.byref(red), per)
        if st != abi.HP_OK:
            msg = (self._lib.hp_multi_last_error(self._m) or b"").decode()
            if st == abi.HP_BAD_CONFIG:
                raise abi.ConfigError(msg)
            raise RuntimeError(f"hp_search_multi failed (status {st}): {msg}")
        return red, list(per)

    def search_log(self) -> List[abi.SearchLogEntry]:
        n, nb = C.c_uint64(), C.c_uint64()
        st = self._lib.hp_multi_search_log(self._m, None, 0, None, 0, C.byref(n), C.byref(nb))
        if st != abi.HP_OK:
            raise RuntimeError((self._lib.hp_multi_last_error(self._m) or b"").decode())
        ents = (abi.hp_log_entry * max(1, n.value))()
        text = C.create_string_buffer(max(1, nb.value))
        st = self._lib.hp_multi_search_log(self._m, ents, n.value, text, nb.value, C.byref(n), C.byref(nb))
        if st != abi.HP_OK:
            raise RuntimeError((self._lib.hp_multi_last_error(self._m) or b"").decode())
        raw = text.raw
        out = []
        for k in range(n.value):
            e = ents[k]
            out.append(abi.SearchLogEntry(raw[e.candidate:raw.index(b"\0", e.candidate)].decode(), e.time_s,
                                          raw[e.reason:raw.index(b"\0", e.reason)].decode()))
        return out


_engines: Dict[int, Engine] = {}


def engine(device: int = 0) -> Engine:
    if device not in _engines:
        _engines[device] = Engine(device)
    return _engines[device]


def _outcome(problem: abi.Problem, res: abi.hp_result) -> SearchOutcome:
    return SearchOutcome(plan=problem.plan_to_doc(res.best_plan), iteration_time_s=res.best_time_s,
                         candidates_simulated=res.candidates_simulated,
                         candidates_pruned=res.candidates_pruned,
                         reason_counts={k: int(res.reason_counts[i]) for i, k in enumerate(abi.REASONS)},
                         device_ms=res.device_ms, gpu_launches=res.gpu_launches, leaves=res.leaves,
                         tasks=res.tasks, global_bound=res.global_bound, raw=res)


def infeasible_reasons(log: List[abi.SearchLogEntry], n_tasks: int) -> List[str]:
    """InfeasibleError reasons of planner.cpp:666-678: the first 200 distinct
    "candidate -> reason" lines of the log."""
    reasons, seen = [], set()
    for e in log:
        if not e.prune_reason:
            continue
        line = e.candidate + " -> " + e.prune_reason
        if line not in seen:
            seen.add(line)
            if len(reasons) < 200:
                reasons.append(line)
    if n_tasks == 0:
        reasons.append("no usable pipeline degree: candidates must lie in [1, num_layers] and fit the "
                       "cluster's node counts")
    return reasons


def merge_logs(parts: List[List[Tuple[int, int, abi.SearchLogEntry]]]) -> List[abi.SearchLogEntry]:
    """Global log from per-shard logs: shards own whole tasks or whole leaves,
    so a stable sort on (task, leaf) restores the reference's order."""
    allp = [x for part in parts for x in part]
    allp.sort(key=lambda x: (x[0], x[1]))
    return [x[2] for x in allp]


def search(docs: Dict[str, dict], jobs: int = 1, device: int = 0, log: bool = False) -> SearchOutcome:
    """search() of planner.hpp:115-116 on one GPU (`jobs` is accepted for
    signature parity; the GPU replaces the thread pool). log=True fills
    SearchOutcome.log; an infeasible search raises InfeasibleError with the
    reference's reason list (taken from the log)."""
    problem = abi.Problem(docs)
    eng = engine(device)
    res = eng.search_shard(problem, flags=abi.HP_FLAG_LOG if log else 0)
    entries = merge_logs([eng.search_log()]) if log else []
    if not res.has_best:
        if not log:
            eng.search_shard(problem, flags=abi.HP_FLAG_LOG)
            entries = merge_logs([eng.search_log()])
        raise abi.InfeasibleError("no feasible plan found", infeasible_reasons(entries, res.tasks))
    out = _outcome(problem, res)
    out.log = entries
    return out


def evaluate_plan(docs: Dict[str, dict], plan: dict, trace: bool = True, device: int = 0) -> PlanEvaluation:
    """evaluate_plan_unchecked(plan, ..., record_trace) (evaluate.hpp:56-58):
    the winner post-processing of search() (planner.cpp:681-684)."""
    problem = abi.Problem(docs)
    return engine(device).evaluate_plan_full(problem, problem.plan_from_doc(plan), trace)


def evaluate_plans(docs: Dict[str, dict], plans: List[dict], device: int = 0) -> List[float]:
    problem = abi.Problem(docs)
    return engine(device).evaluate_plans(problem, [problem.plan_from_doc(p) for p in plans])


def reduce_results(problem: abi.Problem, results: List[abi.hp_result]) -> abi.hp_result:
    """Deterministic reduction of per-shard results: counts add up, the best
    record is picked with the reference's better_than (hp_better_than)."""
    out = abi.hp_result()
    l = lib()
    for r in results:
        out.candidates_simulated += r.candidates_simulated
        out.candidates_pruned += r.candidates_pruned
        for i in range(abi.HP_REASON_COUNT):
            out.reason_counts[i] += r.reason_counts[i]
        out.leaves += r.leaves
        out.tasks = r.tasks
        out.gpu_launches += r.gpu_launches
        out.device_ms = max(out.device_ms, r.device_ms)
        out.global_bound = r.global_bound
        if r.has_best and (not out.has_best or l.hp_better_than(problem.ptr(), r.best_time_s, C.byref(r.best_plan),
                                                                out.best_time_s, C.byref(out.best_plan)) < 0):
            out.has_best = 1
            out.best_time_s = r.best_time_s
            out.best_pp = r.best_pp
            C.memmove(C.byref(out.best_plan), C.byref(r.best_plan), C.sizeof(abi.hp_plan))
    return out


def gather_results(res: abi.hp_result, world: int, group=None, device=None) -> List[abi.hp_result]:
    """All-gathers the fixed-size per-rank hp_result records in one
    collective (NCCL over NVLink with CUDA tensors; gloo with CPU tensors)."""
    import torch
    import torch.distributed as dist

    nbytes = C.sizeof(abi.hp_result)
    dev = f"cuda:{device}" if device is not None else "cpu"
    mine = torch.frombuffer(bytearray(C.string_at(C.byref(res), nbytes)), dtype=torch.uint8).to(dev)
    gathered = torch.empty(world * nbytes, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(gathered, mine, group=group)
    host = gathered.cpu().numpy().tobytes()
    recs = []
    for r in range(world):
        rec = abi.hp_result()
        C.memmove(C.byref(rec), host[r * nbytes:(r + 1) * nbytes], nbytes)
        recs.append(rec)
    return recs


def search_sharded(docs: Dict[str, dict], rank: int, world: int, device: Optional[int] = None, group=None,
                   shard_fn=None, probe_fn=None, log: bool = False, flags: int = 0,
                   mine: Optional[list] = None) -> SearchOutcome:
    """One shard per rank; default mode first all-reduces (MIN) the per-shard
    probe bounds (planner.cpp:640-651), then every rank searches its shard and
    the per-rank records are all-gathered in one collective; every rank
    applies the same exact reduction, so all ranks return the same plan.
    shard_fn/probe_fn replace the GPU engine (tests drive the CPU emulation
    through the same reduction with gloo). `flags` adds HP_FLAG_* bits to
    the shard call; `mine`, if given, receives this rank's own hp_result."""
    import torch
    import torch.distributed as dist

    problem = abi.Problem(docs)
    log_fn = None
    if shard_fn is None:
        eng = engine(device)
        fl = flags | (abi.HP_FLAG_LOG if log else 0)
        shard_fn = lambda p, r, w, b: eng.search_shard(p, r, w, b, fl)  # noqa: E731
        probe_fn = lambda p, r, w: eng.probe_shard(p, r, w)  # noqa: E731
        log_fn = eng.search_log
    bound = None
    if problem.struct.planner.time_bound_pruning and world > 1:
        b = probe_fn(problem, rank, world)
        t = torch.tensor([b], dtype=torch.float64, device=f"cuda:{device}" if device is not None else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        bound = float(t.item())
    res = shard_fn(problem, rank, world, bound)
    if mine is not None:
        mine.append(res)
    red = reduce_results(problem, gather_results(res, world, group, device)) if world > 1 else res
    entries = []
    if log and log_fn is not None:
        parts = [log_fn()]
        if world > 1:
            parts = [None] * world
            dist.all_gather_object(parts, log_fn(), group=group)  # cold path: variable-size log
        entries = merge_logs(parts)
    if not red.has_best:
        raise abi.InfeasibleError("no feasible plan found", infeasible_reasons(entries, red.tasks))
    out = _outcome(problem, red)
    out.log = entries
    return out
