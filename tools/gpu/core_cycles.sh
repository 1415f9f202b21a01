#!/bin/bash
# core-loop cycles per level of the climb kernel's items (HP_DEBUG_TRACE_ITEMS ev 5)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python tools/run_search.py C3 full 1 > /dev/null 2>&1
HP_DEBUG_TRACE=gpurun_out/trace_c3.bin HP_DEBUG_TRACE_ITEMS=1 python tools/run_search.py C3 full 1 > /dev/null 2>&1
python - > gpurun_out/core_cycles.txt 2>&1 <<'PY'
import numpy as np
raw = np.fromfile("gpurun_out/trace_c3.bin", dtype=np.uint64).reshape(-1, 2)
pk = raw[:, 1]
ev = ((pk >> np.uint64(59)) & np.uint64(0xf)).astype(int)
m = ev == 5
cyc = raw[m, 0].astype(np.int64)
P = ((pk[m] >> np.uint64(48)) & np.uint64(0xff)).astype(int)
M = ((pk[m] >> np.uint64(32)) & np.uint64(0xffff)).astype(int)
aux = ((pk[m] >> np.uint64(20)) & np.uint64(0xfff)).astype(int)
lv = 2 * M - 2 - 2 * P
ok = lv > 256
r = cyc[ok] / lv[ok]
print("items", ok.sum(), "cycles/level: min %.1f p10 %.1f median %.1f p90 %.1f" % (r.min(), np.percentile(r, 10), np.median(r), np.percentile(r, 90)))
for p in (12, 24, 48, 96):
    s = ok & (P == p)
    if s.any():
        rr = cyc[s] / lv[s]
        print("P", p, "items", s.sum(), "min %.1f p10 %.1f median %.1f" % (rr.min(), np.percentile(rr, 10), np.median(rr)))
PY
rm -f gpurun_out/trace_c3.bin
