#!/bin/bash
# A/B of tuning builds in paper_2405_16256_b200/_variants/*.so (HP_LIB) on C3 full
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/variant_ab.txt
python tools/run_search.py C3 full 1 > /dev/null 2>&1
for rep in 1 2; do
for v in base $(ls paper_2405_16256_b200/_variants/*.so 2>/dev/null); do
  if [ $v = base ]; then unset HP_LIB; else export HP_LIB=$v; fi
  echo "== $v" >> gpurun_out/variant_ab.txt
  python tools/run_search.py C3 full 3 2>&1 | tail -2 | cut -c1-100 >> gpurun_out/variant_ab.txt
done
done
