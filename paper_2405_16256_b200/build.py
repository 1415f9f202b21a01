"""Builds the in-tree product library libhetplan_b200.so for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false (bit-exact FP64:
no contraction of a*b+c anywhere, SURVEY.md finding 3); host C++ with
-ffp-contract=off for the same reason. The library travels to the GPU box
with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhetplan_b200.so")
OBJ = os.path.join(HERE, "_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "--fmad=false", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
          "-I" + os.path.join(HERE, "..", "include")]
SOURCES = ["hp_kernels.cu", "hp_host.cpp", "hp_log.cpp", "hp_eval.cpp", "hp_capi.cpp", "hp_multi.cpp"]


def _newest_dep_mtime() -> float:
    m = 0.0
    for d in (CSRC, os.path.join(HERE, "..", "include")):
        for f in os.listdir(d):
            m = max(m, os.path.getmtime(os.path.join(d, f)))
    return m


def needs_build() -> bool:
    return not os.path.exists(OUT) or os.path.getmtime(OUT) < _newest_dep_mtime()


def build(verbose: bool = False, ptxas_v: bool = False, out: str = OUT, defines=(), obj_dir: str = OBJ) -> str:
    """defines: extra -D flags (tuning variants, tools/tune/); out/obj_dir
    redirect a variant build away from the product library."""
    os.makedirs(obj_dir, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]

    def compile_one(src):
        obj = os.path.join(obj_dir, src + ".o")
        cmd = [NVCC, *ARCH, *COMMON, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if ptxas_v and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose=True, ptxas_v="-v" in sys.argv))
