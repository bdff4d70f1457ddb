"""Aggregate an ncu --metrics gpu__time_duration.sum csv by kernel name."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', ''))
    v *= {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}.get(r[ui], 1e-6)
    name = r[ki].split('(')[0][:70]
    agg[name][0] += 1; agg[name][1] += v; tot += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.3f} ms {100 * t / tot:5.1f}% {n:6d} avg {1e3 * t / n:9.1f} us  {k}")
print(f"total {tot:.3f} ms, units {rows[hi+1][ui]}")
