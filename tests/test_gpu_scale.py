"""Full-size properties on the B200 (sizes the CPU oracle cannot finish in a
test): the C3 Llama-140B / 768-device full strategy sweep, determinism,
shard-count invariance of the reduction, and agreement with the
time-bound-pruned search (whose C3 outcome is pinned by the reference)."""
from __future__ import annotations

import json
import os

import pytest

from conftest import GOLDEN
from paper_2405_16256_b200 import abi, configs, planner

pytestmark = pytest.mark.gpu

C3_PLAN = ("1f1b|192|1|gpu_a:0-12:8:8:8|gpu_a:12-24:8:8:8|gpu_a:24-36:8:8:8|gpu_a:36-47:8:8:8|gpu_a:47-59:8:8:8|"
           "gpu_a:59-70:8:8:8|gpu_a:70-82:8:8:8|gpu_a:82-94:8:8:8|gpu_a:94-105:8:8:8|gpu_a:105-115:8:8:8|"
           "amd:115-138:8:8:8|amd:138-160:8:8:8")
C3_TIME = 138.65139569127317  # reference, C3 default mode


def test_c3_default_mode_matches_reference_numbers(engine):
    """the reference's C3 default search simulates 1,866 and
    prunes 216,837 candidates and picks pp12 dp8 tp8 M192 at 138.651396 s."""
    p = abi.Problem(configs.config("C3", full=False))
    r = engine.search_shard(p)
    assert (r.candidates_simulated, r.candidates_pruned) == (1866, 216837)
    assert r.best_time_s == C3_TIME
    assert abi.encode_plan(p.group_names, r.best_plan) == C3_PLAN


def test_c3_full_sweep(engine):
    p = abi.Problem(configs.config("C3", full=True))
    a = engine.search_shard(p)
    b = engine.search_shard(p)
    # deterministic, and the full sweep finds the same optimum as the pruned
    # search (the bound is admissible and this instance has no hill-climb
    # divergence at the optimum)
    assert a.best_time_s == b.best_time_s == C3_TIME
    assert abi.encode_plan(p.group_names, a.best_plan) == C3_PLAN
    assert (a.candidates_simulated, a.candidates_pruned) == (b.candidates_simulated, b.candidates_pruned)
    # pinned by the compiled reference itself, one search per pp job
    # (tests/golden/gen_c3_full_ref.py)
    want = json.load(open(os.path.join(GOLDEN, "c3_full_ref.json")))
    assert (a.candidates_simulated, a.candidates_pruned) == (want["candidates_simulated"],
                                                             want["candidates_pruned"])
    assert a.best_time_s == want["best_iteration_time_s"]
    assert abi.encode_plan(p.group_names, a.best_plan) == abi.encode_plan(p.group_names,
                                                                          p.plan_from_doc(want["best_plan"]))


@pytest.mark.parametrize("pps", [[12], [24], [64], [88], [89, 90], [91, 92], [93, 94], [95, 96]])
def test_c3_full_sweep_per_pp_counts(engine, pps):
    """Per-pp slices of the sweep — the long-climb regime (pp 88-96) in
    particular — against the reference's per-pp counts."""
    want = json.load(open(os.path.join(GOLDEN, "c3_full_ref.json")))["per_pp"]
    p = abi.Problem(configs.with_pp(configs.config("C3", full=True), pps))
    r = engine.search_shard(p)
    assert r.candidates_simulated == sum(want[str(x)]["simulated"] for x in pps)
    assert r.candidates_pruned == sum(want[str(x)]["pruned"] for x in pps)


@pytest.mark.parametrize("count", [2, 3, 8])
def test_shard_reduction_invariance(engine, count):
    """N shards on one GPU, reduced exactly, equal the unsharded search
    (what the 8-GPU NCCL path computes)."""
    for full in (True, False):
        docs = configs.with_pp(configs.config("C3", full=full), [10, 12, 20])
        p = abi.Problem(docs)
        whole = engine.search_shard(p)
        bound = None
        if not full:
            bound = min(engine.probe_shard(p, s, count) for s in range(count))
        parts = [engine.search_shard(p, s, count, bound) for s in range(count)]
        red = planner.reduce_results(p, parts)
        assert red.best_time_s == whole.best_time_s
        assert (red.candidates_simulated, red.candidates_pruned) == (whole.candidates_simulated,
                                                                     whole.candidates_pruned)
        assert abi.encode_plan(p.group_names, red.best_plan) == abi.encode_plan(p.group_names, whole.best_plan)


SCHED_KNOBS = [
    {},
    {"HP_CRIT_WARPS": "0"},                      # no critical leaves: rings 1/2 only
    {"HP_HI_LEVELS": "1000000000000"},           # no long-climber ring
    {"HP_NO_LEAD": "1", "HP_NO_LAT": "1"},       # priority ring served by every warp, dense evaluator
    {"HP_CRIT_WARPS": "100000", "HP_HI_LEVELS": "1"},  # (almost) everything prioritised
    {"HP_ASYNC_THREADS": "128"},                 # 4 warps per block
    {"HP_CRIT_SMS": "37"},                       # critical ring on reserved SMs only
    {"HP_CRIT_SMS": "74", "HP_CRIT_MODE": "0"},  # reserved SMs' lead warps also serve bulk
    {"HP_CRIT_SMS": "74", "HP_CRIT_MODE": "2"},  # reserved SMs: critical items only
    {"HP_CRIT_SMS": "148", "HP_R1_THR": "0"},    # every SM reserved; ring 1 on every warp
    {"HP_CRIT_SMS": "148"},                      # every SM reserved: warps 4-7 serve rings 1/2
    {"HP_CRIT_SMS": "148", "HP_CRIT_MODE": "2"},  # (mode 2 falls back to 1: rings 1/2 need servers)
    {"HP_CRIT_SMS": "74", "HP_ASYNC_THREADS": "128"},  # 4-warp blocks: no ring-0-only warps
    {"HP_R1_THR": "100000"},                     # ring 1 on lead warps only
]


@pytest.mark.parametrize("knobs", SCHED_KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
def test_climb_scheduling_does_not_change_results(engine, knobs):
    """The climb kernel's scheduling (critical leaves, priority rings, lead
    warps, latency evaluator, block size; read per search from the
    environment) may only change the order in which items run: counts, time
    and plan must be identical, with and without the search log, on C3
    subsets with long climbs (pp 12 and 88-96)."""
    cfg = configs.with_pp(configs.config("C3", full=True), [12, 88, 92, 96])
    p = abi.Problem(cfg)
    old = {k: os.environ.get(k) for k in knobs}
    os.environ.update(knobs)
    try:
        r = engine.search_shard(p)
        rl = engine.search_shard(p, flags=abi.HP_FLAG_LOG)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ref = engine.search_shard(p)
    # the compiled reference's per-pp counts (tests/golden/c3_full_ref.json)
    want = json.load(open(os.path.join(GOLDEN, "c3_full_ref.json")))["per_pp"]
    sims = sum(want[str(x)]["simulated"] for x in (12, 88, 92, 96))
    prs = sum(want[str(x)]["pruned"] for x in (12, 88, 92, 96))
    for x in (r, rl, ref):
        assert (x.candidates_simulated, x.candidates_pruned) == (sims, prs)
        assert x.best_time_s == ref.best_time_s
        assert abi.encode_plan(p.group_names, x.best_plan) == abi.encode_plan(p.group_names, ref.best_plan)


def test_default_mode_shards_in_fresh_process():
    """A sharded default-mode search as each rank of a multi-GPU run does it,
    in a fresh process (kernel attributes set by no earlier search): probe,
    search with a bound, no error, and every shard's counts add up."""
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2405_16256_b200 import abi, configs, planner\n"
            "eng = planner.engine(0)\n"
            "p = abi.Problem(configs.config('C3', full=False))\n"
            "b = min(eng.probe_shard(p, s, 4) for s in range(4))\n"
            "rs = [eng.search_shard(p, s, 4, b) for s in range(4)]\n"
            "red = planner.reduce_results(p, rs)\n"
            "print(red.candidates_simulated, red.candidates_pruned, repr(red.best_time_s))\n" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    sim, pr, t = out.stdout.split()
    assert (int(sim), int(pr), float(t)) == (1866, 216837, C3_TIME)
