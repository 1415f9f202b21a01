#!/bin/bash
# 1-GPU bench.py A/B of library builds (HP_LIB), alternating
# usage: LIBS="default tools/tune/ab/x.so" ROUNDS=3 bash tools/gpu/bench_lib_ab.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-3}); do
  for l in $LIBS; do
    if [ "$l" = default ]; then e=""; else e="HP_LIB=$l"; fi
    env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bab.json 2> /dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/bab.json').read().strip().splitlines()[-1]); print('$l', round(d['ms_per_step'], 2), round(d['default_mode']['device_ms'], 2))" >> gpurun_out/bench_lib_ab.txt
  done
done
