#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/stage_ab.txt
python tools/run_search.py C3 full 1 > /dev/null 2>&1
for rep in 1 2; do
for v in "HP_X=0" "HP_NO_STAGE=1"; do
  echo "== $v" >> gpurun_out/stage_ab.txt
  env $v python tools/run_search.py C3 full 3 2>&1 | tail -2 | cut -c1-90 >> gpurun_out/stage_ab.txt
  env $v python tools/run_search.py C3 default 3 2>&1 | tail -2 | cut -c1-90 >> gpurun_out/stage_ab.txt
done
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
