#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi2.txt
NCCL_DEBUG=VERSION timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_evaluate.py tests/test_gpu_dropin.py -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_multi.log
