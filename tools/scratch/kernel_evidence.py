"""Summarise ncu per-launch metric CSVs into a per-kernel evidence table:
launches, average duration, achieved DRAM GB/s, DMMA TF/s (m8n8k4 f64 =
512 flop per warp instruction), FP64-pipe active %."""
import csv, collections, sys
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    try:
        hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    except IndexError:
        continue
    h = rows[hi]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value')
    ui = h.index('Metric Unit'); ii = h.index('ID')
    seen = set()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split('(')[0].replace('qtt::', '').replace('<unnamed>::', '')[:48]
        key = (path, r[ii])
        if key not in seen:
            seen.add(key); cnt[name] += 1
        v = float(r[vi].replace(',', '')) if r[vi] not in ('', 'n/a') else 0.0
        unit = r[ui]
        if r[mi] == 'gpu__time_duration.sum':
            v *= {'ns': 1e-9, 'nsecond': 1e-9, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3}.get(unit, 1e-9)
        if r[mi].startswith('dram__bytes'):
            v *= {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)
        agg[name][r[mi]] += v
print(f"{'kernel':48s} {'n':>5s} {'avg us':>9s} {'DRAM GB/s':>10s} {'DMMA TF/s':>10s} {'fp64 pipe%':>10s}")
for name, m in sorted(agg.items(), key=lambda x: -x[1]['gpu__time_duration.sum'])[:30]:
    t = m['gpu__time_duration.sum']; n = cnt[name]
    dram = (m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']) / t / 1e9 if t else 0
    dmma = m['sm__inst_executed_pipe_tensor_subpipe_dmma.sum'] * 512 / t / 1e12 if t else 0
    fp = m['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'] / max(n, 1)
    print(f"{name:48s} {n:5d} {t / n * 1e6:9.1f} {dram:10.1f} {dmma:10.2f} {fp:10.1f}")
