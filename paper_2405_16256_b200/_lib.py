"""Loads the in-tree CUDA library (libhetplan_b200.so). Fails loudly: there is
no CPU fallback for the hot path."""
from __future__ import annotations

import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libhetplan_b200.so")
# tuning builds (tools/tune/) point this at an alternative in-tree build
if os.environ.get("HP_LIB"):
    SO = os.path.abspath(os.environ["HP_LIB"])

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO):
        raise NativeLibraryMissing(
            f"{SO} is missing; build it with `python -m paper_2405_16256_b200.build` "
            "(the CUDA path has no fallback)")
    l = C.CDLL(SO)
    P = C.POINTER
    l.hp_abi_version.restype = C.c_int
    l.hp_create.argtypes = [P(C.c_void_p), C.c_int]
    l.hp_create.restype = C.c_int
    l.hp_destroy.argtypes = [C.c_void_p]
    l.hp_destroy.restype = None
    l.hp_last_error.argtypes = [C.c_void_p]
    l.hp_last_error.restype = C.c_char_p
    l.hp_validate.argtypes = [C.c_void_p, P(abi.hp_problem)]
    l.hp_validate.restype = C.c_int
    l.hp_probe.argtypes = [C.c_void_p, P(abi.hp_problem), P(abi.hp_search_opts), P(C.c_double)]
    l.hp_probe.restype = C.c_int
    l.hp_search.argtypes = [C.c_void_p, P(abi.hp_problem), P(abi.hp_search_opts), P(abi.hp_result)]
    l.hp_search.restype = C.c_int
    l.hp_better_than.argtypes = [P(abi.hp_problem), C.c_double, P(abi.hp_plan), C.c_double, P(abi.hp_plan)]
    l.hp_better_than.restype = C.c_int
    l.hp_evaluate_plans.argtypes = [C.c_void_p, P(abi.hp_problem), P(abi.hp_plan), C.c_int32, P(C.c_double)]
    l.hp_evaluate_plans.restype = C.c_int
    l.hp_search_log.argtypes = [C.c_void_p, P(abi.hp_log_entry), C.c_uint64, C.c_char_p, C.c_uint64,
                                P(C.c_uint64), P(C.c_uint64)]
    l.hp_search_log.restype = C.c_int
    l.hp_evaluate_plan_full.argtypes = [C.c_void_p, P(abi.hp_problem), P(abi.hp_plan), P(abi.hp_plan_eval),
                                        P(abi.hp_stage_eval), P(abi.hp_trace_event), C.c_uint64]
    l.hp_evaluate_plan_full.restype = C.c_int
    l.hp_device_count.restype = C.c_int
    l.hp_multi_create.argtypes = [P(C.c_void_p), P(C.c_int32), C.c_int32]
    l.hp_multi_create.restype = C.c_int
    l.hp_multi_destroy.argtypes = [C.c_void_p]
    l.hp_multi_destroy.restype = None
    l.hp_multi_last_error.argtypes = [C.c_void_p]
    l.hp_multi_last_error.restype = C.c_char_p
    l.hp_search_multi.argtypes = [C.c_void_p, P(abi.hp_problem), C.c_int32, P(abi.hp_result), P(abi.hp_result)]
    l.hp_search_multi.restype = C.c_int
    l.hp_multi_search_log.argtypes = [C.c_void_p, P(abi.hp_log_entry), C.c_uint64, C.c_char_p, C.c_uint64,
                                      P(C.c_uint64), P(C.c_uint64)]
    l.hp_multi_search_log.restype = C.c_int
    if l.hp_abi_version() != abi_version():
        raise NativeLibraryMissing("libhetplan_b200.so ABI version mismatch; rebuild")
    _lib = l
    return l


def abi_version() -> int:
    return 3


EXPORTED = ["hp_abi_version", "hp_create", "hp_destroy", "hp_last_error", "hp_validate", "hp_probe",
            "hp_search", "hp_search_log", "hp_better_than", "hp_evaluate_plans", "hp_evaluate_plan_full",
            "hp_device_count", "hp_multi_create", "hp_multi_destroy", "hp_multi_last_error", "hp_search_multi", "hp_multi_search_log"]
