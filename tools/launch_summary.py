"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
SC = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}
tot = collections.defaultdict(float); cnt = collections.Counter(); mx = collections.defaultdict(float)
for r in data:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', '')) * SC[r[ui]]
    name = r[ki].split('(')[0]
    tot[name] += v; cnt[name] += 1; mx[name] = max(mx[name], v)
allt = sum(tot.values())
print(f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'max ms':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:48]:48s} {cnt[k]:8d} {tot[k]:10.2f} {mx[k]:9.3f} {tot[k]/allt*100:5.1f}%")
print(f"{'sum':48s} {sum(cnt.values()):8d} {allt:10.2f}")
