#!/bin/bash
# A/B timing of tuning variants on the GPU: C3 full sweep, 3 reps each.
# usage: tools/tune/ab.sh name1 name2 ...   (tools/tune/_lib/<name>.so)
for n in "$@"; do
  echo "== $n"
  HP_LIB=tools/tune/_lib/$n.so timeout 600 python tools/run_search.py C3 full 3 2>&1 | tail -3
done
