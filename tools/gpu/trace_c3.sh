#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python tools/run_search.py C3 full 1 > /dev/null 2>&1
HP_DEBUG_TRACE=gpurun_out/trace_c3.bin HP_DEBUG_TRACE_ITEMS=1 python tools/run_search.py C3 full 1 > gpurun_out/trace_run.txt 2>&1
python - > gpurun_out/trace_summary.txt 2>&1 <<'PY'
import numpy as np
raw = np.fromfile("gpurun_out/trace_c3.bin", dtype=np.uint64).reshape(-1, 2)
pk = raw[:, 1]
ev = ((pk >> np.uint64(59)) & np.uint64(0xf)).astype(int)
keep = ev <= 4
raw = raw[keep]; pk = raw[:, 1]; ev = ev[keep]
ns = raw[:, 0].astype(np.int64)
leaf = (pk & np.uint64(0xfffff)).astype(int)
P = ((pk >> np.uint64(48)) & np.uint64(0xff)).astype(int)
M = ((pk >> np.uint64(32)) & np.uint64(0xffff)).astype(int)
aux = ((pk >> np.uint64(20)) & np.uint64(0xfff)).astype(int)
t = (ns - ns.min()) / 1e6
print("records", len(t), "span", t.max())
for e in range(5): print("ev", e, (ev == e).sum(), "first", t[ev == e].min(), "last", t[ev == e].max())
u, c = np.unique(leaf[ev == 0], return_counts=True)
L = int(u[np.argmax(c)])
m = leaf == L
o = np.argsort(t[m], kind="stable")
tt, ee, aa = t[m][o], ev[m][o], aux[m][o]
print("leaf", L, "P", P[m][0], "M", M[m][0], "events", len(tt))
for k in range(min(40, len(tt))): print(f"{tt[k]:9.3f} ev{ee[k]} aux{aa[k]}")
# item starts in first 25 ms by P class
for lo, hi in ((0, 2), (2, 5), (5, 10), (10, 25)):
    s = (ev == 1) & (t >= lo) & (t < hi)
    print(f"items started {lo}-{hi} ms:", s.sum(), "by P>=84:", (s & (P >= 84)).sum())
PY
rm -f gpurun_out/trace_c3.bin
