#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python tools/run_search.py C3 default 3 > gpurun_out/def_times.txt 2>&1
HP_DEBUG_TASKS=gpurun_out/def_tasks.txt python tools/run_search.py C3 default 1 >> gpurun_out/def_times.txt 2>&1
