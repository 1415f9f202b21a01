"""Search-log parity (SearchOutcome::log, planner.hpp:95-107; SURVEY §8f
row 1) through the C ABI: every golden case's log (entry count, SHA-256 of
all entries, first entries verbatim) against the compiled reference's
(tests/golden/search_logs.json), the InfeasibleError reason list
(planner.cpp:666-678), and shard-merged logs equal to the single-device log.
"""
from __future__ import annotations

import hashlib
import struct

import pytest

from conftest import load_golden
from paper_2405_16256_b200 import abi, planner

pytestmark = pytest.mark.gpu


def time_bits(t: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", t))[0]


def rows(entries):
    return [(e.candidate, time_bits(e.time_s), e.prune_reason) for e in entries]


def digest(rs) -> str:
    h = hashlib.sha256()
    for c, b, r in rs:
        h.update(f"{c}\t{b}\t{r}\n".encode())
    return h.hexdigest()


@pytest.fixture(scope="module")
def logs():
    return {c["name"]: c for c in load_golden("search_logs.json")}


def test_logs_match_reference(engine, search_cases, logs):
    checked = 0
    for case in search_cases:
        want = logs[case["name"]]
        if want["status"] != 0:
            continue
        out = planner.search(case["docs"], log=True)
        got = rows(out.log)
        assert got[:len(want["head"])] == [tuple(x) for x in want["head"]], case["name"]
        assert len(got) == want["n"], case["name"]
        assert digest(got) == want["sha256"], case["name"]
        assert len(got) == out.candidates_simulated + out.candidates_pruned
        checked += 1
    assert checked > 100


def test_infeasible_reasons_match_reference(engine, search_cases, logs):
    n = 0
    for case in search_cases:
        want = logs[case["name"]]
        if want["status"] != 2:
            continue
        with pytest.raises(abi.InfeasibleError) as ei:
            planner.search(case["docs"])
        assert ei.value.reasons == want["reasons"], case["name"]
        n += 1
    assert n > 0


@pytest.mark.parametrize("shards", [2, 3])
def test_sharded_logs_merge_to_reference(engine, search_cases, logs, shards):
    picked = [c for c in search_cases if logs[c["name"]]["status"] == 0][:40]
    for case in picked:
        p = abi.Problem(case["docs"])
        bound = None
        if p.struct.planner.time_bound_pruning:
            bound = min(engine.probe_shard(p, k, shards) for k in range(shards))
        parts = []
        for k in range(shards):
            engine.search_shard(p, k, shards, bound, abi.HP_FLAG_LOG)
            parts.append(engine.search_log())
        got = rows(planner.merge_logs(parts))
        assert digest(got) == logs[case["name"]]["sha256"], (case["name"], shards)


def test_log_needs_flag(engine, search_cases):
    p = abi.Problem(search_cases[0]["docs"])
    engine.search_shard(p)
    with pytest.raises(abi.ConfigError):
        engine.search_log()


def test_c3_default_log_matches_reference(engine):
    from paper_2405_16256_b200 import configs
    want = load_golden("c3_default_log.json")
    out = planner.search(configs.config("C3", full=False), log=True)
    got = rows(out.log)
    assert got[:4] == [tuple(x) for x in want["head"]]
    assert len(got) == want["n"]
    assert digest(got) == want["sha256"]


def test_c3_full_log_matches_reference_per_pp(engine):
    """C3 full sweep with the log (10,513,178 entries): for every pipeline
    degree, the entry count, the simulated / pruned split and the SHA-256 of
    that pp's slice of the log equal the compiled reference's, run one pp job
    at a time (tests/golden/gen_c3_full_ref.py; ~36 CPU-hours)."""
    import ctypes as C
    import json as J
    import numpy as np
    from paper_2405_16256_b200 import configs
    want = load_golden("c3_full_ref.json")["per_pp"]
    p = abi.Problem(configs.config("C3", full=True))
    res = engine.search_shard(p, flags=abi.HP_FLAG_LOG)
    n, nb = C.c_uint64(), C.c_uint64()
    assert engine._lib.hp_search_log(engine._ctx, None, 0, None, 0, C.byref(n), C.byref(nb)) == abi.HP_OK
    assert n.value == res.candidates_simulated + res.candidates_pruned == 10513178
    ents = (abi.hp_log_entry * n.value)()
    text = C.create_string_buffer(nb.value)
    assert engine._lib.hp_search_log(engine._ctx, ents, n.value, text, nb.value, C.byref(n), C.byref(nb)) == abi.HP_OK
    e = np.frombuffer(ents, dtype=np.dtype([("c", "<u8"), ("r", "<u8"), ("t", "<f8"), ("task", "<i4"),
                                            ("leaf", "<i4")]))
    raw = text.raw
    cs, rs, tasks = e["c"].tolist(), e["r"].tolist(), e["task"].tolist()
    bl = e["t"].view("<u8").tolist()
    got = {}
    cur_task, pp, h, sim, pru = None, None, None, 0, 0

    def flush():
        if pp is not None:
            d = got.setdefault(pp, [hashlib.sha256(), 0, 0])
            d[0] = h
            d[1] += sim
            d[2] += pru

    for k in range(n.value):
        c0 = cs[k]
        cand = raw[c0:raw.index(b"\0", c0)]
        if tasks[k] != cur_task:
            cur_task = tasks[k]
            npp = J.loads(cand)["pp"]
            if npp != pp:
                flush()
                pp, h, sim, pru = npp, hashlib.sha256(), 0, 0
        r0 = rs[k]
        reason = raw[r0:raw.index(b"\0", r0)]
        h.update(cand + b"\t" + b"%016x" % bl[k] + b"\t" + reason + b"\n")
        if reason:
            pru += 1
        else:
            sim += 1
    flush()
    assert sorted(got) == sorted(int(k) for k in want)
    for pp, (hh, s_, p_) in got.items():
        w = want[str(pp)]
        assert (s_, p_) == (w["simulated"], w["pruned"]), pp
        assert hh.hexdigest() == w["sha256"], pp


def test_c3_full_log_is_complete(engine):
    """C3 full sweep with the log (10.5 M entries; the reference needs ~8 CPU-
    hours for it, so no digest): the replay consumes every GPU time and its
    counts equal the GPU's (checked inside hp_search), one entry per
    candidate."""
    import ctypes as C
    from paper_2405_16256_b200 import configs
    p = abi.Problem(configs.config("C3", full=True))
    res = engine.search_shard(p, flags=abi.HP_FLAG_LOG)
    n = C.c_uint64()
    nb = C.c_uint64()
    assert engine._lib.hp_search_log(engine._ctx, None, 0, None, 0, C.byref(n), C.byref(nb)) == abi.HP_OK
    assert n.value == res.candidates_simulated + res.candidates_pruned == 10513178
