#!/usr/bin/env python3
"""Benchmark of the hot path: the planner's full strategy sweep on C3
(Llama-140B, 768 devices = 128 AMD + 640 accelerator A).

A "step" is one complete search() over the C3 candidate space
(time_bound_pruning = false: every leaf's uniform/proportional seeds plus
its steepest-descent layer-split search, planner.cpp:404-490), ending in the
exact better_than argmin. value = candidates (simulated + pruned, counted like
planner.hpp:101-107) per second of device time, inputs resident (CUDA events
around the device work of each call, max over ranks); e2e = the same through
the public API (planner.search_sharded -> C ABI) with the problem built from
host documents and the result read back, every step. The CLI-default mode
(time_bound_pruning = true) of the same config is timed the same way and
reported under "default_mode". Counts follow the reference
(config.device_work says how many candidates the GPU simulated to the end).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: launched by torchrun, one rank per GPU; ranks take disjoint,
cost-balanced leaf shards and reduce with one NCCL all-gather (strong
scaling: the total sweep is fixed). --impl reference times the compiled,
unmodified reference planner (oracle/_ref) on the host cores, rank 0 only, on a
bounded, work-matched deterministic sample of the same sweep (SAMPLE_DESC).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "candidate plans evaluated/sec (Llama-140B, 768 dev); time-to-optimal-plan"
UNIT = "candidates/s"
WORKLOAD = ("C3: Llama-140B (L=160, H=8192, seq 4096) on 768 devices (amd 16x8 + gpu_a 80x8), "
            "G=1536, B in {1,2}, pp 1..96, full strategy sweep (time_bound_pruning=false)")
# Reference-arm / cpu_baseline sample (the reference needs ~26 CPU-hours for
# the whole sweep, tests/golden/c3_full_ref.json): pipeline degree 64 of the
# same sweep, a complete search of that degree, one micro-batch size per step
# (B = 1 on even steps, 2 on odd ones; both together are the whole pp = 64
# slice: 30,694 candidates). Work per candidate is close to the sweep's: mean
# simulated P*M per candidate 80,968 on pp 64 against 66,314 for the sweep
# (tests/golden/c3_full_counts.json), so the reference's cand/s on the sample
# UNDERSTATES its sweep rate by about that ratio; `cpu_baseline` also carries
# the reference's measured whole-sweep CPU time. The GPU is timed on exactly
# this sample as well (`cpu_baseline.gpu_same_sample`, device and e2e).
CPU_SAMPLE_PP = [64]
CPU_SAMPLE_B = ([1], [2])
WARMUP_PP = [8]  # reference-arm warm-up steps: a cheap slice (untimed)
SAMPLE_DESC = ("work-matched sample of the C3 full sweep: pipeline degree 64, micro-batch 1 (even steps) / 2 "
               "(odd steps); mean simulated P*M per candidate 80,968 vs 66,314 for the whole sweep")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU baseline

def cpu_sample_cfg(step: int = 0, pps=None):
    """The sample of step `step`: pp 64 of the sweep with micro-batch 1
    (even steps) or 2 (odd steps)."""
    from paper_2405_16256_b200 import configs
    cfg = configs.with_pp(configs.config("C3", full=True), pps or CPU_SAMPLE_PP)
    cfg["planner"]["micro_batch_candidates"] = CPU_SAMPLE_B[step % 2]
    return cfg


def run_reference_once(cfg, jobs):
    """The compiled, unmodified reference search() (oracle/_ref), or the C port
    when the reference library is absent. Returns (candidates, seconds, kind)."""
    from oracle import ref
    if ref.available():
        r = ref.search(cfg, jobs=jobs)
        if r.get("status") != 0:
            raise RuntimeError(f"reference search failed: {r.get('error')}")
        return r["candidates_simulated"] + r["candidates_pruned"], r["wall_s"], "reference"
    from oracle import port
    from paper_2405_16256_b200 import abi
    p = abi.Problem(cfg)
    t0 = time.perf_counter()
    st, res = port.search(p)
    return res.candidates_simulated + res.candidates_pruned, time.perf_counter() - t0, "port"


def full_sweep_reference():
    """The reference's measured whole-sweep CPU time (one process per pp
    job, jobs = 1; tests/golden/gen_c3_full_ref.py), when committed."""
    f = os.path.join(HERE, "tests", "golden", "c3_full_ref.json")
    if not os.path.exists(f):
        return None
    d = json.load(open(f))
    cands = d["candidates_simulated"] + d["candidates_pruned"]
    cpu_s = d["reference_cpu_seconds"]
    return {"candidates": cands, "cpu_seconds_1_core": cpu_s, "value_1_core": cands / cpu_s, "unit": UNIT,
            "cpu": d.get("cpu"), "source": "tests/golden/c3_full_ref.json (build container, measured per pp)"}


def cpu_baseline(jobs):
    """One reference step on the sample (micro-batch 1 half: ~10-20 s on 16
    host threads), plus the reference's C3 default-mode search."""
    cfg = cpu_sample_cfg(0)
    cands, secs, kind = run_reference_once(cfg, jobs)
    out = {"value": cands / secs, "unit": UNIT, "cores": jobs if kind == "reference" else 1, "kind": kind,
           "sample": f"C3 full sweep, pipeline degree {CPU_SAMPLE_PP}, micro-batch {CPU_SAMPLE_B[0]} "
                     f"({cands} candidates, {secs:.2f} s)"}
    from paper_2405_16256_b200 import configs
    dc, ds, _ = run_reference_once(configs.config("C3", full=False), jobs)
    out["default_mode"] = {"time_to_plan_s": ds, "candidates": dc,
                           "workload": "C3 default mode (time_bound_pruning=true), whole search"}
    fs = full_sweep_reference()
    if fs:
        out["full_sweep"] = fs
    return out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ reference arm

def main_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    jobs = os.cpu_count() or 1
    for _ in range(args.warmup):  # untimed: a cheap slice warms the process
        run_reference_once(cpu_sample_cfg(0, WARMUP_PP), jobs)
    cands_all, secs_all, kind = 0, 0.0, None
    for k in range(args.steps):
        cands, secs, kind = run_reference_once(cpu_sample_cfg(k), jobs)
        cands_all += cands
        secs_all += secs
    ms = secs_all / args.steps * 1e3
    value = cands_all / secs_all
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "sample": SAMPLE_DESC,
                       "candidates_per_step": cands_all / args.steps, "cpu": cpu_model(), "threads": jobs},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": jobs if kind == "reference" else 1,
                             "kind": kind, "sample": SAMPLE_DESC},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    fs = full_sweep_reference()
    if fs:
        line["cpu_baseline"]["full_sweep"] = fs
    emit(line)
    return 0


# ------------------------------------------------------------------ our arm

def main_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2405_16256_b200 import abi, configs, planner
    from paper_2405_16256_b200._lib import lib

    rank, world, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one rank per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    docs = configs.config(args.config, full=True)
    docs_default = configs.config(args.config, full=False)
    problem = abi.Problem(docs)

    def one_step(d, flags=0):
        """One complete search through the public API (planner.search_sharded:
        host documents -> C ABI -> sm_100a kernels -> per-rank result -> one
        NCCL all-gather -> exact reduction; default mode adds the NCCL MIN
        all-reduce of the probe bounds). Returns (outcome, this rank's record)."""
        mine = []
        out = planner.search_sharded(d, rank, world, device=local, flags=flags, mine=mine)
        return out, mine[0]

    # L2 flush buffer (> 126 MB L2) written between timed steps
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def timed(d, steps, warmup, clk=None):
        for _ in range(warmup):
            one_step(d)
        torch.cuda.synchronize()
        rec = {"dev_ms": [], "wall_ms": [], "eval_ms": 0.0, "eval_ops": 0.0, "launches": 0, "h2d": 0.0,
               "d2h": 0.0, "dsim": 0, "dabort": 0, "dscreen": 0}
        out = None
        for _ in range(steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            out, mine = one_step(d, abi.HP_FLAG_TIME_KERNELS)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if world > 1:
                dist.barrier()
            rec["dev_ms"].append(mine.device_ms)
            rec["wall_ms"].append((t1 - t0) * 1e3)
            rec["eval_ms"] += mine.eval_ms
            rec["eval_ops"] += mine.eval_fp64_ops
            rec["launches"] = mine.gpu_launches
            rec["h2d"], rec["d2h"] = mine.h2d_bytes, mine.d2h_bytes
            rec["dsim"], rec["dabort"], rec["dscreen"] = mine.device_simulated, mine.device_aborted, \
                mine.device_screened
        torch.cuda.synchronize()
        # max over ranks of the per-step times; sums of bytes/launches/work over ranks
        vec = torch.tensor([sum(rec["dev_ms"]) / steps, sum(rec["wall_ms"]) / steps], dtype=torch.float64,
                           device="cuda")
        agg = torch.tensor([rec["h2d"], rec["d2h"], float(rec["launches"]), rec["eval_ms"], rec["eval_ops"],
                            float(rec["dsim"]), float(rec["dabort"]), float(rec["dscreen"])],
                           dtype=torch.float64, device="cuda")
        per_rank = [float(vec[0])]
        if world > 1:
            allv = torch.empty(world * 2, dtype=torch.float64, device="cuda")
            dist.all_gather_into_tensor(allv, vec)
            per_rank = [float(x) for x in allv[0::2].cpu()]
            dist.all_reduce(vec, op=dist.ReduceOp.MAX)
            dist.all_reduce(agg, op=dist.ReduceOp.SUM)
        return out, float(vec[0]), float(vec[1]), [float(x) for x in agg], per_rank

    with ClockSampler(local) as clk:
        out, dev_step_ms, wall_step_ms, agg, per_rank = timed(docs, args.steps, args.warmup)
    h2d, d2h, launches, eval_ms_all, eval_ops_all, dsim, dabort, dscreen = agg
    # CLI-default mode (time_bound_pruning = true) of the same config: a
    # complete search with its own time to plan, same contract
    dout, ddev_ms, dwall_ms, dagg, _ = timed(docs_default, args.steps, args.warmup)

    cands = out.candidates_simulated + out.candidates_pruned
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    l = lib()
    l.hp_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    dadd, mix = C.c_double(), C.c_double()
    l.hp_fp64_peak(local, C.byref(dadd), C.byref(mix))
    achieved = eval_ops_all / (eval_ms_all * 1e-3) if eval_ms_all > 0 else None
    peak = dadd.value
    traffic = None
    tf = os.path.join(HERE, "profiles", "latest_eval_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    dcands = dout.candidates_simulated + dout.candidates_pruned
    line = {
        "metric": METRIC, "value": cands / (dev_step_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "time_to_plan_s": wall_step_ms / 1e3,
        "config": {"workload": WORKLOAD, "candidates_per_step": cands,
                   "candidates_simulated": out.candidates_simulated, "candidates_pruned": out.candidates_pruned,
                   "count_semantics": ("candidates as the reference counts them (planner.hpp:101-107): every "
                                       "candidate the reference decides; device_work says how many the GPU "
                                       "simulated to the end"),
                   "device_work": {
                       "simulated_to_end": int(dsim), "aborted_by_bound": int(dabort),
                       "screened_by_bound": int(dscreen),
                       "simulated_per_s": dsim / (dev_step_ms / 1e3),
                       "note": ("screened/aborted candidates have an admissible lower bound above the "
                                "current hill-climb point, so they can neither be the move nor tie the leaf "
                                "best; the reference simulates them and so do its counts")},
                   "best_iteration_time_s": out.iteration_time_s,
                   "best_plan": abi.encode_plan(problem.group_names, out.raw.best_plan),
                   "parallelism": f"leaf-sharded x{world}",
                   "rank_device_ms": per_rank,
                   "l2": "flushed between timed steps (256 MiB write); per-step inputs are KB-sized tables"},
        "default_mode": {"workload": "same config, time_bound_pruning=true (CLI default, json_io.cpp:215)",
                         "candidates_per_step": dcands, "candidates_simulated": dout.candidates_simulated,
                         "device_ms": ddev_ms, "time_to_plan_s": dwall_ms / 1e3,
                         "value": dcands / (ddev_ms / 1e3), "e2e_value": dcands / (dwall_ms / 1e3),
                         "best_iteration_time_s": dout.iteration_time_s,
                         "best_plan": abi.encode_plan(problem.group_names, dout.raw.best_plan)},
        "e2e": {"value": cands / (wall_step_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp64", "achieved": achieved / 1e12 if achieved else None,
                     "peak": peak / 1e12, "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic,
                     "note": ("algorithmic FP64 add+max ops of the evaluator kernels (8PM-4M per candidate "
                              "simulated to the end, the levels run for an aborted one) / their CUDA-event "
                              "time; peak = measured DADD rate on this GPU "
                              f"({peak / 1e12:.2f} T/s); the add/max node-update mix peaks at "
                              f"{mix.value / 1e12:.2f} T/s on the same GPU")},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(os.cpu_count() or 1)
            cb["cpu"] = cpu_model()
            # this GPU on exactly the CPU sample, device time and end to end
            sd = cpu_sample_cfg(0)
            sp = abi.Problem(sd)
            one_step(sd)
            t0 = time.perf_counter()
            so, smine = one_step(sd, abi.HP_FLAG_TIME_KERNELS)
            swall = time.perf_counter() - t0
            sc = so.candidates_simulated + so.candidates_pruned
            cb["gpu_same_sample"] = {"value": sc / (smine.device_ms / 1e3), "e2e_value": sc / swall,
                                     "unit": UNIT, "device_ms": smine.device_ms, "e2e_ms": swall * 1e3,
                                     "candidates": sc}
            line["cpu_baseline"] = cb
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the process's original stdout."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # Libraries (NCCL's version banner, CUDA, the engine) may write to fd 1;
    # send all of that to stderr so stdout carries only the JSON line.
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return main_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
