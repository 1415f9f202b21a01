#!/bin/bash
# A/B timing of runtime tuning knobs on the GPU (C3 full sweep, best of 3).
# usage: tools/tune/env_sweep.sh "ENV=.. ENV2=.." "ENV=.." ...
cfg=${CFG:-C3}
for e in "$@"; do
  echo "== $e"
  env $e timeout 600 python tools/run_search.py $cfg full 3 2>&1 | tail -2 | python -c '
import sys, json
rows = [json.loads(l) for l in sys.stdin if l.startswith("{")]
print("  dev_ms", [round(r["dev_ms"], 1) for r in rows], "t", rows[-1]["t"] if rows else None)'
done
