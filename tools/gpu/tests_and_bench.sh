#!/bin/bash
# -m gpu suite + smoke, then a 1-GPU bench (driver settings) and a 4-GPU-free
# quick A/B of a build-time knob when AB_FLAGS is set (tools/gpu/variant_ab.sh)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
bash tools/gpu/full_tests.sh
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench rc=$?" >> gpurun_out/bench_n1.err
