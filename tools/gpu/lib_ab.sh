#!/bin/bash
# A/B of library builds (HP_LIB) on one search config, alternating variants
# usage: CFG=C3:96 LIBS="default tools/tune/ab/u1.so" REPS=3 bash tools/gpu/lib_ab.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
  for l in $LIBS; do
    if [ "$l" = default ]; then
      python tools/run_search.py ${CFG:-C3} full ${REPS:-3} 2>/dev/null | tail -n +2 | python -c "
import sys, json; v=[json.loads(x)['dev_ms'] for x in sys.stdin]; print('$l', '${CFG:-C3}', [round(x,2) for x in v])" >> gpurun_out/lib_ab.txt
    else
      HP_LIB=$l python tools/run_search.py ${CFG:-C3} full ${REPS:-3} 2>/dev/null | tail -n +2 | python -c "
import sys, json; v=[json.loads(x)['dev_ms'] for x in sys.stdin]; print('$l', '${CFG:-C3}', [round(x,2) for x in v])" >> gpurun_out/lib_ab.txt
    fi
  done
done
