"""TEST INFRASTRUCTURE ONLY: ctypes handle on the plain-C restatement
(oracle/hetplan_oracle.c -> oracle/_build/libhetplan_oracle.so). Used by
tests/ as the checker and by bench.py's cpu_baseline leg ("port")."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2405_16256_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libhetplan_oracle.so")


class ho_leaf_info(C.Structure):
    _fields_ = [("task", C.c_int32), ("pp", C.c_int32), ("dp", C.c_int32), ("tp", C.c_int32 * abi.HP_MAX_GROUPS),
                ("B", C.c_int64), ("M", C.c_int64), ("exhaustive", C.c_int32), ("hill_steps", C.c_int32),
                ("evaluated", C.c_int64), ("simulated", C.c_int64), ("pruned", C.c_int64)]


LEAF_CB = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(ho_leaf_info))

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            build()
        l = C.CDLL(SO)
        l.ho_search.argtypes = [C.POINTER(abi.hp_problem), C.POINTER(abi.hp_result), LEAF_CB, C.c_void_p]
        l.ho_search.restype = C.c_int
        l.ho_evaluate.argtypes = [C.POINTER(abi.hp_problem), C.POINTER(abi.hp_plan), C.POINTER(C.c_double)]
        l.ho_evaluate.restype = C.c_int
        l.ho_simulate.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int64, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]
        l.ho_simulate.restype = C.c_int
        l.ho_split_layers.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int)]
        l.ho_split_layers.restype = C.c_int
        _lib = l
    return _lib


def search(problem: abi.Problem, leaf_cb=None):
    res = abi.hp_result()
    cb = LEAF_CB(lambda u, li: leaf_cb(li.contents)) if leaf_cb else LEAF_CB()
    st = lib().ho_search(C.byref(problem.struct), C.byref(res), cb, None)
    return st, res


def evaluate(problem: abi.Problem, plan: abi.hp_plan) -> float:
    out = C.c_double()
    rc = lib().ho_evaluate(C.byref(problem.struct), C.byref(plan), C.byref(out))
    if rc:
        raise ValueError("oracle evaluate failed")
    return out.value


def simulate(times, M, gpipe=False):
    P = len(times)
    flat = (C.c_double * (4 * P))(*[x for t in times for x in t])
    it = C.c_double()
    ce = (C.c_double * P)()
    rc = lib().ho_simulate(int(gpipe), flat, P, M, C.byref(it), ce)
    if rc:
        raise ValueError("oracle simulate rejected input")
    return it.value, list(ce)


def split_layers(total, weights):
    n = len(weights)
    out = (C.c_int * max(1, n))()
    rc = lib().ho_split_layers(total, (C.c_double * max(1, n))(*weights), n, out)
    if rc == 1:
        raise ValueError("ConfigError")
    if rc == 2:
        raise ArithmeticError("InfeasibleError")
    return list(out)[:n]
