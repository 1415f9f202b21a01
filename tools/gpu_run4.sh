#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python tools/run_search.py C3 default 4 > gpurun_out/def_times.txt 2>&1
HP_DEBUG_TASKS=gpurun_out/def_tasks.txt python tools/run_search.py C3 default 1 >> gpurun_out/def_times.txt 2>&1
python tools/run_search.py C3 full 3 >> gpurun_out/def_times.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
