"""Winner post-processing (planner.cpp:681-684) through
the C ABI (hp_evaluate_plan_full): the full PlanEvaluation of
evaluate_plan_unchecked(record_trace = true) (evaluate.cpp:78-107) — stage
costs, busy times, compute ends, bubble ratios, retained activations, peak
memory and the sorted trace (sim.cpp:63-209) — bit for bit against the
compiled reference (oracle/_ref), on every golden winner and on random
explicit plans."""
from __future__ import annotations

import random
import struct

import pytest

from conftest import load_golden
from oracle import ref
from paper_2405_16256_b200 import abi, configs, planner

pytestmark = pytest.mark.gpu


def bits(x: float) -> str:
    return struct.pack(">d", x).hex()


def check(docs, plan_doc, name):
    want = ref.evaluate_trace(docs, plan_doc)
    assert want["status"] == 0, (name, want.get("error"))
    w = want["eval"]
    got = planner.evaluate_plan(docs, plan_doc, trace=True)
    ev = got.eval
    assert bits(ev.iteration_time_s) == w["iteration_bits"], name
    assert bits(ev.pipeline_time_s) == w["pipeline_bits"], name
    assert bits(ev.aggregate_bubble_ratio) == w["aggregate_bubble_bits"], name
    assert ev.micro_batches == w["micro_batches"] and ev.total_devices == w["total_devices"], name
    assert ev.n_stages == len(w["stages"]), name
    for i, (s, ws) in enumerate(zip(got.stages, w["stages"])):
        for ours, theirs in (("fwd_s", "fwd"), ("bwd_s", "bwd"), ("send_fwd_s", "send_fwd"),
                             ("send_bwd_s", "send_bwd"), ("dp_sync_s", "dp_sync"), ("compute_end_s", "compute_end"),
                             ("busy_s", "busy"), ("bubble_ratio", "bubble"), ("peak_memory_bytes", "peak_memory")):
            assert bits(getattr(s, ours)) == ws[theirs], (name, i, ours)
        assert s.peak_in_flight == ws["peak_in_flight"], (name, i)
    assert len(got.trace) == len(w["trace"]), name
    for e, we in zip(got.trace, w["trace"]):
        assert [e.stage, e.kind, e.microbatch, bits(e.start_s), bits(e.end_s)] == we, name


def test_golden_winners_post_processing(search_cases):
    n = 0
    for case in search_cases:
        if case["status"] != 0:
            continue
        check(case["docs"], case["plan"], case["name"])
        n += 1
    for case in load_golden("c4_c5_cases.json"):
        if case["status"] == 0:
            check(case["docs"], case["plan"], case["name"])
            n += 1
    assert n > 150


def test_c3_winner_post_processing():
    docs = configs.config("C3", full=False)
    out = planner.search(docs)
    check(docs, out.plan, "C3")


def test_random_plans_post_processing():
    """GPipe and 1F1B, M < P and M >= P, mixed groups / tp / dp."""
    rng = random.Random(11)
    docs = configs.config("C0", full=True)
    L = docs["model"]["num_layers"]
    p = abi.Problem(docs)
    for k in range(60):
        P = min(L, rng.choice([1, 2, 3, 5, 8, 12, 20, 40]))
        cuts = sorted(rng.sample(range(1, L), P - 1))
        bounds = [0] + cuts + [L]
        pl = abi.hp_plan()
        pl.schedule = rng.choice([0, 1])
        pl.micro_batches_per_dp_replica = rng.choice([1, 2, 3, 7, 16, 64])
        pl.micro_batch_size = rng.choice([0, 1, 2])
        pl.n_stages = P
        for i in range(P):
            s = pl.stages[i]
            s.layer_begin, s.layer_end = bounds[i], bounds[i + 1]
            s.group = rng.choice([0, 1])
            s.tp_degree = rng.choice([1, 2, 4, 8])
            s.dp_degree = rng.choice([1, 2, 4])
            s.nodes_used = rng.choice([1, 2])
        check(docs, p.plan_to_doc(pl), f"random {k}")


def test_plan_shape_rejected():
    docs = configs.config("C0", full=True)
    p = abi.Problem(docs)
    pl = abi.hp_plan()
    pl.schedule = 1
    pl.micro_batches_per_dp_replica = 4
    pl.n_stages = 2
    pl.stages[0].layer_begin, pl.stages[0].layer_end = 0, 10
    pl.stages[1].layer_begin, pl.stages[1].layer_end = 12, docs["model"]["num_layers"]  # gap
    for s in (pl.stages[0], pl.stages[1]):
        s.tp_degree = s.dp_degree = s.nodes_used = 1
    with pytest.raises(abi.ConfigError, match="does not continue"):
        planner.engine(0).evaluate_plan_full(p, pl)


def test_large_plans_gpipe_and_1f1b():
    """GPipe and 1F1B at P*M >= 1e5 (the generic counter-driven evaluator and
    the closed-form 1F1B one): batched iteration times (hp_evaluate_plans)
    and the full evaluation with trace, against the reference."""
    rng = random.Random(23)
    docs = configs.config("C3", full=True)
    L = docs["model"]["num_layers"]
    p = abi.Problem(docs)
    plans = []
    for k in range(8):
        P = rng.choice([64, 80, 96])
        M = rng.choice([1600, 2048])
        cuts = sorted(rng.sample(range(1, L), P - 1))
        bounds = [0] + cuts + [L]
        pl = abi.hp_plan()
        pl.schedule = k % 2  # gpipe, 1f1b alternating
        pl.micro_batches_per_dp_replica = M
        pl.micro_batch_size = 1
        pl.n_stages = P
        for i in range(P):
            s = pl.stages[i]
            s.layer_begin, s.layer_end = bounds[i], bounds[i + 1]
            s.group = 0 if i < P // 5 else 1
            s.tp_degree = 8
            s.dp_degree = 1
            s.nodes_used = 1
        assert P * M >= 1e5
        plans.append(pl)
    times = planner.engine(0).evaluate_plans(p, plans)
    for k, pl in enumerate(plans):
        doc = p.plan_to_doc(pl)
        want = ref.evaluate(docs, doc)["eval"]["iteration_bits"]
        assert bits(times[k]) == want, k
        if k < 4:
            check(docs, doc, f"large {k}")
