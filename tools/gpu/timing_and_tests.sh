#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
HP_DEBUG_TIMING=1 python tools/run_search.py C3 default 4 > gpurun_out/timing.txt 2>&1
HP_DEBUG_TIMING=1 python tools/run_search.py C3 full 3 >> gpurun_out/timing.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_log.py::test_c3_full_log_matches_reference_per_pp -k "not per_pp and not test_c3_full_sweep" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
