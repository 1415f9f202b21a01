"""Shared fixtures. GPU tests are marked @pytest.mark.gpu; everything else
runs on CPU (oracle vs golden vectors, host logic, ABI, gloo multi-process)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
EMU_SO = os.path.join(ROOT, "tests", "emu", "_build", "libemu.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (runs on the B200 box)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def search_cases():
    return load_golden("search_cases.json")


@pytest.fixture(scope="session")
def oracle_port():
    from oracle import port
    port.lib()
    return port


def build_emu():
    src = [os.path.join(ROOT, "tests", "emu", "emu_search.cpp"),
           os.path.join(ROOT, "paper_2405_16256_b200", "csrc", "hp_host.cpp")]
    hdrs = [os.path.join(ROOT, "paper_2405_16256_b200", "csrc", f) for f in
            ("hp_core.cuh", "hp_search_core.cuh", "hp_host.hpp")] + [os.path.join(ROOT, "include", "hetplan_b200.h")]
    newest = max(os.path.getmtime(x) for x in src + hdrs)
    if not os.path.exists(EMU_SO) or os.path.getmtime(EMU_SO) < newest:
        os.makedirs(os.path.dirname(EMU_SO), exist_ok=True)
        subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", EMU_SO] + src,
                       check=True)
    import ctypes as C
    from paper_2405_16256_b200 import abi
    lib = C.CDLL(EMU_SO)
    lib.emu_search.argtypes = [C.POINTER(abi.hp_problem), C.POINTER(abi.hp_result)]
    lib.emu_search_shard.argtypes = [C.POINTER(abi.hp_problem), C.c_int, C.c_int, C.POINTER(abi.hp_result)]
    lib.emu_screen_stats.argtypes = [C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.c_int]
    lib.emu_split_layers.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int)]
    return lib


@pytest.fixture(scope="session")
def emu():
    return build_emu()


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def engine():
    if not gpu_available():
        pytest.skip("no CUDA device")
    from paper_2405_16256_b200 import planner
    return planner.engine(0)
