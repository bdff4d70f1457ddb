# Per-superstep timing of the config-3 TT-SVD: ncu launch durations (cold) + small-phase cycle counts.
QTT_TTSVD_DEBUG=1 python tools/ttsvd_profile.py 2>&1 | grep "ttsvd\]" | tail -30 | cut -c1-220
ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "ttsvd/" --log-file gpurun_out/ttsvd_launches.csv python tools/ttsvd_profile.py > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/ttsvd_launches.csv')))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
tot = 0
for r in rows[hi+1:]:
    if len(r) > vi:
        v = float(r[vi].replace(',', '')) / 1e3; tot += v
        print(f"{v:9.1f} us  {r[ki][:50]}")
print("total us", tot)
PY
