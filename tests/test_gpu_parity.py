"""Parity of the sm_100a search path (through the C ABI) with the reference:
golden outcomes of the compiled reference (tests/golden), seeded random
instances against the C restatement, explicit-plan evaluation bit for bit,
error behaviour. Everything runs on cuda:0."""
from __future__ import annotations

import random
import struct

import pytest

from paper_2405_16256_b200 import abi, configs, planner
from instances import random_instance

pytestmark = pytest.mark.gpu


def hexbits(x):
    return struct.pack(">d", x).hex()


def check_case(engine, case):
    p = abi.Problem(case["docs"])
    if case["status"] == 2:
        res = engine.search_shard(p)
        assert not res.has_best, case["name"]
        with pytest.raises(abi.InfeasibleError):
            planner.search(case["docs"])
        return
    res = engine.search_shard(p)
    assert res.has_best, case["name"]
    assert hexbits(res.best_time_s) == case["iteration_bits"], case["name"]
    assert (res.candidates_simulated, res.candidates_pruned) == (
        case["candidates_simulated"], case["candidates_pruned"]), case["name"]
    want = abi.encode_plan(p.group_names, p.plan_from_doc(case["plan"]))
    assert abi.encode_plan(p.group_names, res.best_plan) == want, case["name"]
    assert res.gpu_launches > 0


def test_golden_cases_both_modes(engine, search_cases):
    for case in search_cases:
        check_case(engine, case)


def test_random_instances_vs_oracle(engine, oracle_port):
    rng = random.Random(99)
    for k in range(80):
        docs = random_instance(rng, k)
        p = abi.Problem(docs)
        st, want = oracle_port.search(p)
        got = engine.search_shard(p)
        if st == abi.HP_INFEASIBLE:
            assert not got.has_best
            continue
        assert got.has_best
        assert got.best_time_s == want.best_time_s, k
        assert (got.candidates_simulated, got.candidates_pruned) == (want.candidates_simulated,
                                                                     want.candidates_pruned), k
        assert abi.encode_plan(p.group_names, got.best_plan) == abi.encode_plan(p.group_names, want.best_plan), k


@pytest.mark.parametrize("full", [True, False])
def test_c3_pipeline_subsets(engine, oracle_port, full):
    """Llama-140B / 768 devices at pp in {8, 12, 16}: large M, K=2..8 lanes."""
    docs = configs.with_pp(configs.config("C3", full=full), [8, 12, 16])
    p = abi.Problem(docs)
    st, want = oracle_port.search(p)
    got = engine.search_shard(p)
    assert got.best_time_s == want.best_time_s
    assert (got.candidates_simulated, got.candidates_pruned) == (want.candidates_simulated, want.candidates_pruned)
    assert abi.encode_plan(p.group_names, got.best_plan) == abi.encode_plan(p.group_names, want.best_plan)


def test_gpipe_and_short_pipelines(engine, oracle_port):
    """Generic evaluator classes: GPipe and M < P."""
    docs = configs.with_pp(configs.config("C0", full=True), [6, 12])
    docs["planner"]["schedule"] = "gpipe"
    docs["model"]["num_layers"] = 24
    for g in docs["cluster"]["groups"]:
        g["memory_bytes"] = 1e18  # GPipe retains all M activations
    for d in (docs,):
        p = abi.Problem(d)
        st, want = oracle_port.search(p)
        got = engine.search_shard(p)
        assert st == abi.HP_OK and got.has_best
        assert got.best_time_s == want.best_time_s
        assert (got.candidates_simulated, got.candidates_pruned) == (want.candidates_simulated,
                                                                     want.candidates_pruned)
    short = configs.config("C1", full=True)
    short["train"]["global_batch_size"] = 8  # M = 8/(dp*B) < P for deep pipelines
    p = abi.Problem(short)
    st, want = oracle_port.search(p)
    got = engine.search_shard(p)
    assert got.best_time_s == want.best_time_s
    assert (got.candidates_simulated, got.candidates_pruned) == (want.candidates_simulated, want.candidates_pruned)


def test_evaluate_plans_bit_exact(engine, oracle_port):
    """hp_evaluate_plans == evaluate_plan_unchecked(...).iteration_time_s of
    the compiled reference (and of the C restatement)."""
    rng = random.Random(5)
    docs = configs.config("C0", full=True)
    p = abi.Problem(docs)
    plans = []
    for _ in range(300):
        P = rng.choice([1, 2, 3, 5, 8, 12, 20, 33, 40, 70])
        L = docs["model"]["num_layers"]
        if P > L:
            P = L
        cuts = sorted(rng.sample(range(1, L), P - 1))
        bounds = [0] + cuts + [L]
        pl = abi.hp_plan()
        pl.schedule = rng.choice([0, 1])
        pl.micro_batches_per_dp_replica = rng.choice([1, 2, 3, 7, 16, 64, 200])
        pl.micro_batch_size = rng.choice([0, 1, 2])
        pl.n_stages = P
        for i in range(P):
            s = pl.stages[i]
            s.layer_begin, s.layer_end = bounds[i], bounds[i + 1]
            s.group = rng.choice([0, 1])
            s.tp_degree = rng.choice([1, 2, 4, 8])
            s.dp_degree = rng.choice([1, 2, 4])
            s.nodes_used = rng.choice([1, 2])
        plans.append(pl)
    got = engine.evaluate_plans(p, plans)
    from oracle import ref
    for pl, g in zip(plans, got):
        assert g == oracle_port.evaluate(p, pl)
        want = ref.evaluate(docs, p.plan_to_doc(pl))["eval"]["iteration_bits"]
        assert hexbits(g) == want


def test_bad_config_raises_config_error(engine):
    docs = configs.config("C0")
    docs["model"]["num_heads"] = 7
    with pytest.raises(abi.ConfigError, match="divisible by num_heads"):
        planner.search(docs)


def test_c4_c5_against_reference(engine):
    """SURVEY §8d C4 (all six accelerator pairs, Llama-70B / 512 devices;
    default mode over every pp with the search log, full mode on pp
    {2..12}) and C5 (pp 3 exhaustive slices, 160 layers, 3 device types)
    against the compiled reference's outcomes (tests/golden/gen_c4_c5.py)."""
    import hashlib
    from conftest import load_golden
    cases = load_golden("c4_c5_cases.json")
    assert sum(c["name"].startswith("C4:") for c in cases) == 12
    assert any(c["name"].startswith("C5:") and c["status"] == 0 for c in cases)
    for case in cases:
        check_case(engine, case)
        if "log" in case:
            out = planner.search(case["docs"], log=True)
            h = hashlib.sha256()
            for e in out.log:
                h.update(f"{e.candidate}\t{struct.pack('>d', e.time_s).hex()}\t{e.prune_reason}\n".encode())
            assert len(out.log) == case["log"]["n"], case["name"]
            assert h.hexdigest() == case["log"]["sha256"], case["name"]


def test_climb_cases_against_reference(engine):
    """60 full-sweep instances where the hill climb does the work and slow
    (often cpu-staged) links join the groups, so the neighbour screen's
    per-stage and pair-circuit bounds skip most neighbours: plan, time bits
    and counts equal the compiled reference's (tests/golden/gen_climb_cases.py)."""
    from conftest import load_golden
    cases = load_golden("climb_cases.json")["cases"]
    assert len(cases) == 60 and sum(c["status"] == 0 for c in cases) >= 50
    for case in cases:
        check_case(engine, case)


def test_gpipe_search_at_scale(engine):
    """GPipe search at P*M up to 98,304 (C3, pp 64, micro-batch 1, memory
    unbounded): the generic evaluator in the climb kernel against the
    reference's outcome (tests/golden/gen_gpipe_scale.py)."""
    from conftest import load_golden
    case = load_golden("gpipe_scale.json")
    assert case["status"] == 0 and case["candidates_simulated"] > 50000
    check_case(engine, case)
