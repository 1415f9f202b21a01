"""Dev tool: per-step latency breakdown of one leaf from an HP_DEBUG_TRACE
file recorded with HP_DEBUG_TRACE_ITEMS=1 (events: 0 step done, 1 item
start, 2 item end, 3 screened, 4 pushed; hp_kernels.cu: trace_event).
usage: python tools/analysis/item_trace.py trace.bin [leaf]
"""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
ns = raw[:, 0].astype(np.int64)
pk = raw[:, 1]
ev = ((pk >> np.uint64(59)) & np.uint64(0xf)).astype(int)
aux = ((pk >> np.uint64(20)) & np.uint64(0xfff)).astype(int)
leaf = (pk & np.uint64(0xfffff)).astype(int)
P = ((pk >> np.uint64(48)) & np.uint64(0xff)).astype(int)
if len(sys.argv) > 2:
    L = int(sys.argv[2])
else:  # the leaf with the most steps
    u, c = np.unique(leaf[ev == 0], return_counts=True)
    L = int(u[np.argmax(c)])
m = leaf == L
t = (ns[m] - ns[m].min()) / 1e3  # us
e = ev[m]
a = aux[m]
o = np.argsort(t, kind="stable")
t, e, a = t[o], e[o], a[o]
print(f"leaf {L} P {P[m][0]}: steps {np.sum(e == 0)}, items {np.sum(e == 1)}, span {t.max() / 1e3:.2f} ms")
# walk: step boundaries are ev 0 (step done) ... ev 3 screened, ev 4 pushed, items, last item end, ev 0
rows = []
i = 0
n = len(t)
last0 = None
cur = {}
for k in range(n):
    if e[k] == 0:
        if "t0" in cur and cur.get("push") is not None and cur.get("ends"):
            rows.append((cur["t0"], cur["scr"], cur["push"], min(cur["starts"]), max(cur["starts"]),
                         max(cur["ends"]), t[k], cur["n"], np.mean(np.array(cur["ends"]) - np.array(cur["starts"][:len(cur["ends"])]))))
        cur = {"t0": t[k], "starts": [], "ends": []}
    elif e[k] == 3:
        cur["scr"] = t[k]
        cur["n"] = a[k]
    elif e[k] == 4:
        cur["push"] = t[k]
    elif e[k] == 1:
        cur.setdefault("starts", []).append(t[k])
    elif e[k] == 2:
        cur.setdefault("ends", []).append(t[k])
r = np.array(rows)
if len(r):
    print("mean us: step->screened %.1f, screened->pushed %.1f, pushed->first start %.1f, first->last start %.1f, "
          "item dur %.1f, last end->step done %.1f, total/step %.1f, survivors %.1f" % (
              np.mean(r[:, 1] - r[:, 0]), np.mean(r[:, 2] - r[:, 1]), np.mean(r[:, 3] - r[:, 2]),
              np.mean(r[:, 4] - r[:, 3]), np.mean(r[:, 8]), np.mean(r[:, 6] - r[:, 5]),
              np.mean(r[:, 6] - r[:, 0]), np.mean(r[:, 7])))
    # by step index quartile (the history scan grows with the step count)
    q = np.array_split(np.arange(len(r)), 4)
    print("last end->step done by quartile of the climb (us):",
          [round(float(np.mean(r[ix, 6] - r[ix, 5])), 1) for ix in q])
    print("item dur by quartile (us):", [round(float(np.mean(r[ix, 8])), 1) for ix in q])
