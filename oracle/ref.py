"""TEST INFRASTRUCTURE ONLY: ctypes handle on the compiled, unmodified
reference planner (oracle/_ref/libhetplan_ref.so, built by oracle/Makefile
from /root/reference/proj/core/src). Used by tests/, smoke() and bench.py's
reference leg as the checker / CPU baseline — never by the product path.
"""
from __future__ import annotations

import ctypes
import json
import os
import struct
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libhetplan_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        l = ctypes.CDLL(REF_SO)
        cp = ctypes.c_char_p
        l.ref_search_json.argtypes = [cp, cp, cp, cp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        l.ref_search_json.restype = ctypes.c_int
        l.ref_evaluate_json.argtypes = [cp, cp, cp, cp, ctypes.POINTER(ctypes.c_void_p)]
        l.ref_evaluate_json.restype = ctypes.c_int
        l.ref_evaluate_trace_json.argtypes = [cp, cp, cp, cp, ctypes.POINTER(ctypes.c_void_p)]
        l.ref_evaluate_trace_json.restype = ctypes.c_int
        l.ref_simulate.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                   ctypes.c_longlong, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_double)]
        l.ref_simulate.restype = ctypes.c_int
        l.ref_split_layers.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int)]
        l.ref_split_layers.restype = ctypes.c_int
        l.ref_calibrate_json.argtypes = [cp, cp, cp, ctypes.POINTER(ctypes.c_void_p)]
        l.ref_calibrate_json.restype = ctypes.c_int
        l.ref_free.argtypes = [ctypes.c_void_p]
        _lib = l
    return _lib


def _take(p: ctypes.c_void_p) -> dict:
    s = ctypes.string_at(p.value).decode()
    lib().ref_free(p)
    return json.loads(s)


def bits_to_float(h: str) -> float:
    return struct.unpack("<d", bytes.fromhex(h)[::-1])[0]


def search(cfg: dict, jobs: int = 1, want_log: bool = False) -> dict:
    out = ctypes.c_void_p()
    enc = [json.dumps(cfg[k]).encode() for k in ("model", "cluster", "train", "planner")]
    lib().ref_search_json(*enc, jobs, int(want_log), ctypes.byref(out))
    return _take(out)


def evaluate(cfg: dict, plan: dict) -> dict:
    out = ctypes.c_void_p()
    enc = [json.dumps(cfg[k]).encode() for k in ("model", "cluster", "train")] + [json.dumps(plan).encode()]
    lib().ref_evaluate_json(*enc, ctypes.byref(out))
    return _take(out)


def evaluate_trace(cfg: dict, plan: dict) -> dict:
    """evaluate_plan_unchecked(record_trace=true): every PlanEvaluation field
    as bits plus the sorted trace."""
    out = ctypes.c_void_p()
    enc = [json.dumps(cfg[k]).encode() for k in ("model", "cluster", "train")] + [json.dumps(plan).encode()]
    lib().ref_evaluate_trace_json(*enc, ctypes.byref(out))
    return _take(out)


def calibrate(model: dict, cluster: dict, profiles_text: str) -> dict:
    out = ctypes.c_void_p()
    lib().ref_calibrate_json(json.dumps(model).encode(), json.dumps(cluster).encode(),
                             profiles_text.encode(), ctypes.byref(out))
    return _take(out)


def simulate(times, M: int, gpipe: bool = False):
    """times: list of (fwd, bwd, send_fwd, send_bwd). Returns (iteration, compute_end list)."""
    P = len(times)
    flat = (ctypes.c_double * (4 * P))(*[x for t in times for x in t])
    it = ctypes.c_double()
    ce = (ctypes.c_double * P)()
    rc = lib().ref_simulate(int(gpipe), flat, P, M, ctypes.byref(it), ce)
    if rc:
        raise ValueError("ref simulate rejected input")
    return it.value, list(ce)


def split_layers(total: int, weights) -> Optional[list]:
    n = len(weights)
    w = (ctypes.c_double * n)(*weights)
    out = (ctypes.c_int * n)()
    rc = lib().ref_split_layers(total, w, n, out)
    if rc == 1:
        raise ValueError("ConfigError")
    if rc == 2:
        raise ArithmeticError("InfeasibleError")
    return list(out)
