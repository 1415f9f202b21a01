"""Multi-GPU search inside the C ABI (hp_multi_*, NCCL between the GPUs of
one process; planner.cpp:612-664): on 2+ GPUs the reduced result equals the
single-GPU search bit for bit (counts, time, plan, and the merged search
log), in both pruning modes. Needs >= 2 GPUs (gpurun --gpus 2); skipped
otherwise."""
from __future__ import annotations

import pytest

from conftest import load_golden
from paper_2405_16256_b200 import abi, configs, planner

pytestmark = pytest.mark.gpu


def n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.fixture(scope="module")
def multi():
    n = n_gpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    m = planner.MultiEngine(list(range(n)))
    yield m
    m.close()


def same(a, b, p):
    assert (a.candidates_simulated, a.candidates_pruned) == (b.candidates_simulated, b.candidates_pruned)
    assert a.best_time_s == b.best_time_s
    assert abi.encode_plan(p.group_names, a.best_plan) == abi.encode_plan(p.group_names, b.best_plan)


@pytest.mark.parametrize("full", [True, False])
def test_multi_equals_single_c3(multi, engine, full):
    p = abi.Problem(configs.config("C3", full=full))
    red, per = multi.search(p)
    one = engine.search_shard(p)
    same(red, one, p)
    assert len(per) == len(multi.devices) and all(r.gpu_launches > 0 for r in per)
    assert red.device_ms == max(r.device_ms for r in per)


def test_multi_log_and_golden_cases(multi, search_cases):
    logs = {c["name"]: c for c in load_golden("search_logs.json")}
    import hashlib
    import struct
    n = 0
    for case in search_cases[:60]:
        if case["status"] != 0:
            continue
        p = abi.Problem(case["docs"])
        red, _ = multi.search(p, abi.HP_FLAG_LOG)
        assert struct.pack(">d", red.best_time_s).hex() == case["iteration_bits"], case["name"]
        assert (red.candidates_simulated, red.candidates_pruned) == (case["candidates_simulated"],
                                                                     case["candidates_pruned"]), case["name"]
        h = hashlib.sha256()
        for e in multi.search_log():
            h.update(f"{e.candidate}\t{struct.pack('>d', e.time_s).hex()}\t{e.prune_reason}\n".encode())
        assert h.hexdigest() == logs[case["name"]]["sha256"], case["name"]
        n += 1
    assert n > 30


def test_dropin_jobs_selects_gpus(multi, search_cases):
    """The drop-in's `jobs` (planner.hpp:115-116) picks that many GPUs
    (hp_search_multi): same outcome and log as the reference."""
    import ctypes
    import json
    import os
    from conftest import ROOT
    so = os.path.join(ROOT, "integration", "_build", "libhetplan_dropin.so")
    l = ctypes.CDLL(so)
    cp = ctypes.c_char_p
    l.ref_search_json.argtypes = [cp, cp, cp, cp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    l.ref_free.argtypes = [ctypes.c_void_p]
    for case in search_cases[:30]:
        out = ctypes.c_void_p()
        enc = [json.dumps(case["docs"][k]).encode() for k in ("model", "cluster", "train", "planner")]
        l.ref_search_json(*enc, len(multi.devices), 0, ctypes.byref(out))
        r = json.loads(ctypes.string_at(out.value).decode())
        l.ref_free(out)
        assert r["status"] == case["status"], case["name"]
        if case["status"] == 0:
            assert r["eval"]["iteration_bits"] == case["iteration_bits"], case["name"]
            assert r["plan"] == case["plan"], case["name"]
            assert (r["candidates_simulated"], r["candidates_pruned"]) == (
                case["candidates_simulated"], case["candidates_pruned"]), case["name"]
