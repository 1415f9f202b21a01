"""Dev tool: per-loop stall breakdown from `ncu --page source --csv` (SASS
view) of one kernel: innermost loops (backward branches with no loop inside),
their instruction mix and warp-stall samples by reason.
usage: python tools/analysis/ncu_loops.py src.csv [top]
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        a = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    samp = {k: float(r[ix[k]] or 0) for k in reasons}
    ins.append((a, r[ix["Source"]], float(r[ix["Warp Stall Sampling (All Samples)"]] or 0), samp,
                float(r[ix["Instructions Executed"]] or 0)))
addr = {a: k for k, (a, *_rest) in enumerate(ins)}
total = sum(x[2] for x in ins)
tot_r = Counter()
for x in ins:
    tot_r.update(x[3])
print(f"total samples {total:.0f}; by reason:",
      ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in tot_r.most_common(8)))
loops = []
for k, (a, src, *_r) in enumerate(ins):
    m = re.search(r"BRA\s.*?(0x[0-9a-f]+)", src)
    if m and int(m.group(1), 16) <= a and int(m.group(1), 16) in addr:
        loops.append((addr[int(m.group(1), 16)], k))
inner = [L for L in loops if not any(L[0] <= M[0] and M[1] <= L[1] and M != L for M in loops)]
out = []
for s0, s1 in inner:
    body = ins[s0:s1 + 1]
    samp = sum(x[2] for x in body)
    c = Counter()
    for x in body:
        c.update(x[3])
    nd = sum(1 for x in body if "DADD" in x[1])
    execs = max(x[4] for x in body)
    out.append((samp, hex(ins[s0][0]), len(body), nd, execs, c))
out.sort(key=lambda x: -x[0])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
acc = 0
for samp, a, n, nd, execs, c in out[:top]:
    acc += samp
    print(f"{a}: {n:4d} instr, {nd:3d} DADD, iters {execs:10.0f}, samples {samp / total:6.1%} | " +
          ", ".join(f"{k[6:]} {v / max(samp, 1):.0%}" for k, v in c.most_common(4)))
print(f"top {top} innermost loops: {acc / total:.1%} of samples")
