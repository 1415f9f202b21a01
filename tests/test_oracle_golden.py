"""The C restatement (oracle/hetplan_oracle.c) against golden vectors produced
by the compiled reference (tests/golden/gen_golden.py): search outcomes in
both pruning modes, split_layers and simulate — bit-exact."""
from __future__ import annotations

import struct

import pytest

from conftest import load_golden
from paper_2405_16256_b200 import abi


def hexbits(x: float) -> str:
    return struct.pack(">d", x).hex()


def test_search_cases_match_reference(search_cases, oracle_port):
    assert len(search_cases) >= 150
    for case in search_cases:
        p = abi.Problem(case["docs"])
        st, res = oracle_port.search(p)
        if case["status"] == 2:
            assert st == abi.HP_INFEASIBLE, case["name"]
            continue
        assert st == abi.HP_OK, case["name"]
        assert hexbits(res.best_time_s) == case["iteration_bits"], case["name"]
        assert res.candidates_simulated == case["candidates_simulated"], case["name"]
        assert res.candidates_pruned == case["candidates_pruned"], case["name"]
        want = abi.encode_plan(p.group_names, p.plan_from_doc(case["plan"]))
        assert abi.encode_plan(p.group_names, res.best_plan) == want, case["name"]


def test_readme_sample_counts(search_cases):
    """Survey §6: the shipped sample in default mode simulates 151 and prunes
    521 candidates; the full sweep 1076 / 190 (reproduced by the reference)."""
    by = {c["name"]: c for c in search_cases}
    assert (by["C0-default"]["candidates_simulated"], by["C0-default"]["candidates_pruned"]) == (151, 521)
    assert (by["C0-full"]["candidates_simulated"], by["C0-full"]["candidates_pruned"]) == (1076, 190)
    assert by["C0-default"]["iteration_time_s"] == by["C0-full"]["iteration_time_s"]


def test_split_layers_golden(oracle_port):
    for s in load_golden("split_layers.json"):
        assert oracle_port.split_layers(s["total"], s["w"]) == s["out"]


def test_split_layers_published_fixtures(oracle_port):
    # test_planner.cpp:114-121
    assert oracle_port.split_layers(80, [1.0] * 10) == [8] * 10
    assert oracle_port.split_layers(10, [2.0, 1.0, 1.0]) == [5, 3, 2]
    assert oracle_port.split_layers(7, [1.0, 1.0]) == [4, 3]
    assert oracle_port.split_layers(3, [100.0, 1.0, 1.0]) == [1, 1, 1]
    with pytest.raises(ArithmeticError):
        oracle_port.split_layers(2, [1.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        oracle_port.split_layers(4, [1.0, -1.0])


def test_simulate_golden(oracle_port):
    for s in load_golden("simulate.json"):
        it, ce = oracle_port.simulate(s["times"], s["M"], s["gpipe"])
        assert float(it).hex() == s["iteration_bits"]
        assert ce == s["compute_end"]


def test_simulate_closed_forms(oracle_port):
    # test_sim.cpp:81-126 and acceptance criterion 2
    for P in range(1, 9):
        for M in range(1, 17):
            it, _ = oracle_port.simulate([(0.75, 1.5, 0.0, 0.0)] * P, M)
            assert it == pytest.approx((M + P - 1) * 2.25, rel=1e-12)
    it, _ = oracle_port.simulate([(1.0, 1.0, 0.5, 0.5)] * 2, 1)
    assert it == pytest.approx(5.0)
    it, _ = oracle_port.simulate([(1.0, 2.0, 0.0, 0.0)], 4)
    assert it == pytest.approx(12.0)
