#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/variants.txt
run() { echo "== $*" >> gpurun_out/variants.txt; env "$@" python tools/run_search.py C3 full 2 2>&1 | tail -1 | cut -c1-90 >> gpurun_out/variants.txt; }
python tools/run_search.py C3 full 1 > /dev/null 2>&1
for rep in 1 2; do
run HP_X=0
run HP_CRIT_WARPS=1200
run HP_CRIT_WARPS=2400
run HP_CRIT_WARPS=4800
run HP_R0_THR=64
run HP_R0_THR=64 HP_CRIT_WARPS=2400
run HP_R0_THR=0 HP_CRIT_WARPS=2400
run HP_R0_THR=0 HP_CRIT_WARPS=4800
run HP_CRIT_SMS=32
run HP_CRIT_SMS=48 HP_CRIT_WARPS=1200
run HP_NO_LEAD=1 HP_CRIT_WARPS=4800
done
