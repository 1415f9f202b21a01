"""Builds tuning variants of the product library (compile-time -D knobs)
into tools/tune/ab/<name>.so (git-ignored, travels with gpurun) for A/B
timing on the GPU (tools/gpu/lib_ab.sh, tools/gpu/bench_lib_ab.sh):

    python tools/tune/build_variants.py name1=DEF1,DEF2 name2=...
    HP_LIB=tools/tune/ab/name1.so python tools/run_search.py C3 full 3
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2405_16256_b200 import build  # noqa: E402

OUT = os.path.join(ROOT, "tools", "tune", "ab")


def one(spec):
    name, _, defs = spec.partition("=")
    defines = [d for d in defs.split(",") if d]
    so = os.path.join(OUT, f"{name}.so")
    build.build(out=so, defines=defines, obj_dir=os.path.join(OUT, "_obj_" + name))
    return so


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    with ThreadPoolExecutor(max_workers=4) as ex:
        for so in ex.map(one, sys.argv[1:]):
            print(so)
