"""Dev tool: busy fraction of the sampled climb-kernel warps over time from
an HP_DEBUG_TRACE file recorded with HP_DEBUG_TRACE_ITEMS=n (item start /
end events of every n-th warp; hp_kernels.cu: trace_event).
usage: python tools/analysis/busy.py trace.bin n_sampled_warps
"""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
ns = raw[:, 0].astype(np.int64)
pk = raw[:, 1]
ev = ((pk >> np.uint64(59)) & np.uint64(0xf)).astype(int)
cls = ((pk >> np.uint64(56)) & np.uint64(0x7)).astype(int)
t = (ns - ns.min()) / 1e6
nw = int(sys.argv[2])
m = (ev == 1) | (ev == 2)
tt, ee = t[m], ev[m]
o = np.argsort(tt, kind="stable")
tt, ee = tt[o], ee[o]
d = np.where(ee == 1, 1, -1)
busy = np.cumsum(d)  # warps inside an item
span = t.max()
bins = np.linspace(0, span, 21)
print(f"span {span:.1f} ms, item events {m.sum()}")
for a, b in zip(bins[:-1], bins[1:]):
    sel = (tt >= a) & (tt < b)
    if sel.sum() < 2:
        print(f"{a:7.1f}-{b:7.1f} ms: -")
        continue
    # time-weighted mean of busy over the bin
    x = tt[sel]
    y = busy[sel]
    w = np.diff(np.append(x, b))
    print(f"{a:7.1f}-{b:7.1f} ms: busy {np.sum(y * w) / (b - a) / nw:6.1%}")
