#!/bin/bash
# A/B of environment knobs on C3 full, 1 GPU: KNOBS="A=1 B=2 ..." (one run set each, plus the default)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/knob_ab.txt
python tools/run_search.py C3 full 1 > /dev/null 2>&1
for rep in 1 2; do
for v in HP_X=0 $KNOBS; do
  echo "== $v" >> gpurun_out/knob_ab.txt
  env $v python tools/run_search.py C3 full 3 2>&1 | tail -2 | cut -c1-100 >> gpurun_out/knob_ab.txt
done
done
