"""Dev tool: summarise an HP_DEBUG_TRACE file of a full-mode search.

Each record is (globaltimer ns, packed) with packed = cls<<56 | P<<48 |
M<<32 | move<<20 | leaf (hp_kernels.cu: advance_leaf). Prints per-class
spans, the leaves whose climbs end last, and how many leaves are still
climbing over time (the tail that bounds the class kernels).
usage: python tools/analysis/trace_summary.py trace.bin
"""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
raw = raw[((raw[:, 1] >> np.uint64(59)) & np.uint64(0xf)) == 0]  # step events only
ns = raw[:, 0].astype(np.int64)
pk = raw[:, 1]
t = (ns - ns.min()) / 1e6  # ms
cls = ((pk >> np.uint64(56)) & np.uint64(0x7)).astype(int)
P = ((pk >> np.uint64(48)) & np.uint64(0xff)).astype(int)
M = ((pk >> np.uint64(32)) & np.uint64(0xffff)).astype(int)
leaf = (pk & np.uint64(0xfffff)).astype(int)
print(f"steps recorded: {len(t)}, span {t.max():.2f} ms")
for c in sorted(set(cls)):
    m = cls == c
    print(f"class {c}: steps {m.sum():7d} leaves {len(set(leaf[m])):6d} first {t[m].min():7.2f} "
          f"last {t[m].max():7.2f} ms")
# per leaf: first/last step, number of steps
order = np.lexsort((t, leaf))
lf_s, idx = np.unique(leaf[order], return_index=True)
ends = np.append(idx[1:], len(order))
rows = []
for l, a, e in zip(lf_s, idx, ends):
    sel = order[a:e]
    rows.append((t[sel].max(), t[sel].min(), e - a, P[sel[0]], M[sel[0]], cls[sel[0]], l))
rows.sort(reverse=True)
print("last-finishing leaves: end_ms start_ms steps P M cls leaf  (ms/step)")
for r in rows[:25]:
    per = (r[0] - r[1]) / max(r[2] - 1, 1)
    print(f"  {r[0]:8.2f} {r[1]:8.2f} {r[2]:5d} {r[3]:3d} {r[4]:5d} {r[5]} {r[6]:6d}  ({per:.3f})")
ends_arr = np.array([r[0] for r in rows])
tot = t.max()
print("leaves still climbing at fraction of span:")
for f in (0.25, 0.5, 0.6, 0.7, 0.8, 0.9, 0.95):
    print(f"  {f:.2f} ({f * tot:7.2f} ms): {(ends_arr > f * tot).sum()}")
# step throughput over time (10 bins)
h, e = np.histogram(t, bins=10)
print("steps per 10% of span:", h.tolist())
