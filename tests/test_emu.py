"""CPU emulation of the GPU search decomposition (tests/emu drives the exact
per-candidate / per-leaf device functions of hp_search_core.cuh in loops)
against the reference's golden outcomes: level-synchronous simulator,
on-device seed splits, memo-equivalent hill-climb counting, exhaustive
enumeration order and the encode_plan tie-break, all in full-sweep mode."""
from __future__ import annotations

import ctypes as C
import struct

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
