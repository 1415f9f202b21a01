"""CPU emulation of the GPU search decomposition (tests/emu drives the exact
per-candidate / per-leaf device functions of hp_search_core.cuh in loops)
against the reference's golden outcomes: level-synchronous simulator,
on-device seed splits, memo-equivalent hill-climb counting, exhaustive
enumeration order and the encode_plan tie-break, all in full-sweep mode."""
from __future__ import annotations

import ctypes as C
import struct

import pytest

from paper_2405_16256_b200 import abi


def hexbits(x):
    return struct.pack(">d", x).hex()


def full_cases(search_cases):
    return [c for c in search_cases if not c["docs"]["planner"].get("time_bound_pruning", True)]


def test_emu_matches_reference_full_mode(search_cases, emu):
    """Includes the neighbour screen (nb_screen): neighbours whose path lower
    bound exceeds the current time are not simulated; the C3 pp=12 case
    screens out most of them and must still match the reference exactly."""
    sk, nn = C.c_longlong(), C.c_longlong()
    emu.emu_screen_stats(C.byref(sk), C.byref(nn), 1)
    n = 0
    for case in full_cases(search_cases):
        p = abi.Problem(case["docs"])
        res = abi.hp_result()
        st = emu.emu_search(C.byref(p.struct), C.byref(res))
        if case["status"] == 2:
            assert st == abi.HP_INFEASIBLE, case["name"]
            continue
        assert st == abi.HP_OK, case["name"]
        assert hexbits(res.best_time_s) == case["iteration_bits"], case["name"]
        assert (res.candidates_simulated, res.candidates_pruned) == (
            case["candidates_simulated"], case["candidates_pruned"]), case["name"]
        want = abi.encode_plan(p.group_names, p.plan_from_doc(case["plan"]))
        assert abi.encode_plan(p.group_names, res.best_plan) == want, case["name"]
        n += 1
    assert n >= 60
    emu.emu_screen_stats(C.byref(sk), C.byref(nn), 1)
    assert sk.value > 0.3 * nn.value, (sk.value, nn.value)
    # the screen from precomputed count -1 / +1 stage rows (nb_screen_pre, the
    # GPU's) decides exactly like the per-neighbour stage_setup one
    emu.emu_screen_mismatches.restype = C.c_longlong
    assert emu.emu_screen_mismatches() == 0
    # and the bound never exceeds a simulated time
    emu.emu_bound_violations.restype = C.c_longlong
    assert emu.emu_bound_violations() == 0


def test_emu_screen_is_admissible(search_cases, emu):
    """Every neighbour the screen skips (per-stage and pair-circuit bounds,
    hp_search_core.cuh) is simulated anyway here: its time is never below
    its bound, and it is strictly above the climb point, so skipping it
    cannot change a move, a tie or a count."""
    emu.emu_check_all.restype = C.c_longlong
    emu.emu_bound_violations.restype = C.c_longlong
    before = emu.emu_check_all(1)
    v0 = emu.emu_bound_violations()
    try:
        for case in full_cases(search_cases):
            if case["status"] == 2:
                continue
            p = abi.Problem(case["docs"])
            res = abi.hp_result()
            assert emu.emu_search(C.byref(p.struct), C.byref(res)) == abi.HP_OK
            assert hexbits(res.best_time_s) == case["iteration_bits"], case["name"]
    finally:
        checked = emu.emu_check_all(0) - before
    assert checked > 1000
    assert emu.emu_bound_violations() == v0


def test_emu_climb_cases_screen(emu):
    """The climb-heavy, slow-link instances (tests/golden/climb_cases.json):
    the emulated GPU search equals the reference, the pair-circuit term
    screens neighbours the per-stage bound keeps, and every screened
    neighbour, simulated anyway, is strictly worse than the climb point."""
    from conftest import load_golden
    emu.emu_check_all.restype = C.c_longlong
    emu.emu_bound_violations.restype = C.c_longlong
    sk, nn = C.c_longlong(), C.c_longlong()
    emu.emu_screen_stats(C.byref(sk), C.byref(nn), 1)
    before = emu.emu_check_all(1)
    v0 = emu.emu_bound_violations()
    n = 0
    try:
        for case in load_golden("climb_cases.json")["cases"]:
            p = abi.Problem(case["docs"])
            res = abi.hp_result()
            st = emu.emu_search(C.byref(p.struct), C.byref(res))
            if case["status"] != 0:
                assert st != abi.HP_OK, case["name"]
                continue
            assert st == abi.HP_OK, case["name"]
            assert hexbits(res.best_time_s) == case["iteration_bits"], case["name"]
            assert (res.candidates_simulated, res.candidates_pruned) == (
                case["candidates_simulated"], case["candidates_pruned"]), case["name"]
            n += 1
    finally:
        checked = emu.emu_check_all(0) - before
    emu.emu_screen_stats(C.byref(sk), C.byref(nn), 1)
    assert n >= 50
    assert emu.emu_bound_violations() == v0
    # 129,096 of 899,094 neighbours with the per-stage bound alone
    assert checked == sk.value and sk.value > 200000, (checked, sk.value, nn.value)


def test_emu_shards_partition_the_leaves(search_cases, emu):
    """Leaf shards are disjoint and cover the space: per-shard counts add up
    and the exact reduction (hp_better_than) picks the unsharded plan."""
    from paper_2405_16256_b200 import planner
    cases = [c for c in full_cases(search_cases) if c["status"] == 0]
    for case in cases[:25]:
        p = abi.Problem(case["docs"])
        for count in (2, 3, 5):
            recs = []
            for s in range(count):
                r = abi.hp_result()
                assert emu.emu_search_shard(C.byref(p.struct), s, count, C.byref(r)) == abi.HP_OK
                recs.append(r)
            red = planner.reduce_results(p, recs)
            assert red.candidates_simulated == case["candidates_simulated"]
            assert red.candidates_pruned == case["candidates_pruned"]
            assert hexbits(red.best_time_s) == case["iteration_bits"]
            want = abi.encode_plan(p.group_names, p.plan_from_doc(case["plan"]))
            assert abi.encode_plan(p.group_names, red.best_plan) == want


def test_device_split_layers_matches_reference(emu):
    """hp_core.cuh split_layers (the device apportionment of k_seeds /
    k_default, planner.cpp:42-84) equals the compiled reference on random
    weights: few distinct values (the grouped stable-sort path: stages of a
    device group share a weight) and many (the insertion-sort fallback)."""
    import ctypes as C
    import random
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(17)
    for k in range(3000):
        parts = rng.choice([1, 2, 3, 5, 8, 12, 24, 40, 80, 96, 160])
        total = parts + rng.randrange(0, 400)
        if k % 3 == 0:
            w = [rng.uniform(0.1, 10.0) for _ in range(parts)]
        else:
            vals = [rng.choice([36.0, 94.0, 147.0 * 0.327 * 8, 383 * 0.245 * 4, 1.0]) for _ in range(rng.randint(1, 3))]
            w = [rng.choice(vals) for _ in range(parts)]
            if k % 2:
                s = sum(w)
                w = [x / s for x in w]  # stage_weights normalises (planner.cpp:94-103)
        arr = (C.c_double * parts)(*w)
        out = (C.c_int * parts)()
        emu.emu_split_layers(total, arr, parts, out)
        assert list(out) == ref.split_layers(total, w), (total, w)
