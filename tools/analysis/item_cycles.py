"""Dev tool: evaluator cycle records (HP_DEBUG_TRACE_ITEMS, ev 5 core loop /
ev 6 whole item; hp_kernels.cu: trace_cycles) -> cycles per level.
usage: python tools/analysis/item_cycles.py trace.bin
"""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
pk = raw[:, 1]
ev = ((pk >> np.uint64(59)) & np.uint64(0xf)).astype(int)
P = ((pk >> np.uint64(48)) & np.uint64(0xff)).astype(int)
M = ((pk >> np.uint64(32)) & np.uint64(0xffff)).astype(int)
aux = ((pk >> np.uint64(20)) & np.uint64(0xfff)).astype(int)
cyc = raw[:, 0].astype(np.int64)
c5, c6 = ev == 5, ev == 6
core_levels = (2 * M - 2) - 2 * P + 1
tot_levels = 2 * (M + P - 1)
print(f"core records {c5.sum()} (no-channel-max {np.sum(aux[c5] == 1)}), item records {c6.sum()}")
for k in sorted(set(aux[c6])):
    m6 = c6 & (aux == k)
    print(f"K={k}: items {m6.sum()}, cycles/level whole item median {np.median(cyc[m6] / tot_levels[m6]):.1f}")
ok = c5 & (core_levels > 0)
print(f"core loop cycles/level median {np.median(cyc[ok] / core_levels[ok]):.1f}, "
      f"p10 {np.percentile(cyc[ok] / core_levels[ok], 10):.1f}, p90 {np.percentile(cyc[ok] / core_levels[ok], 90):.1f}")
