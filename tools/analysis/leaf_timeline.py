"""Dev tool: step-time timeline of the longest climbs in an HP_DEBUG_TRACE
file (ms per step in consecutive windows of the leaf's life, next to the
number of leaves still climbing at that time).
usage: python tools/analysis/leaf_timeline.py trace.bin [n_leaves]
"""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
raw = raw[((raw[:, 1] >> np.uint64(59)) & np.uint64(0xf)) == 0]
t = (raw[:, 0].astype(np.int64) - raw[:, 0].astype(np.int64).min()) / 1e6
leaf = (raw[:, 1] & np.uint64(0xfffff)).astype(int)
u, c = np.unique(leaf, return_counts=True)
last = {l: t[leaf == l].max() for l in u}
ends = np.array(sorted(last.values()))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for l in u[np.argsort(-c)][:n]:
    tt = np.sort(t[leaf == l])
    print(f"leaf {l}: {len(tt)} steps, {tt[0]:.1f} -> {tt[-1]:.1f} ms")
    for a in range(0, len(tt) - 1, max(1, len(tt) // 10)):
        b = min(len(tt) - 1, a + max(1, len(tt) // 10))
        alive = (ends > tt[a]).sum()
        print(f"   steps {a:4d}-{b:4d} at {tt[a]:7.1f} ms: {(tt[b] - tt[a]) / (b - a):.3f} ms/step, {alive} leaves climbing")
