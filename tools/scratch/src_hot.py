"""Per-CUDA-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Warp Stall Sampling (All Samples)' in r][0]
h = rows[hi]; si = h.index('Warp Stall Sampling (All Samples)')
agg = collections.Counter(); src = {}; cur = None
for r in rows[hi + 1:]:
    if len(r) <= si: continue
    if r[0].strip():
        cur = r[0]; src[cur] = r[1][:110]
    try: v = float(r[si])
    except ValueError: v = 0.0
    if cur: agg[cur] += v
tot = sum(agg.values()) or 1
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{100 * v / tot:5.1f}% {k:>6} {src[k]}")
