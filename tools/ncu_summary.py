"""Key per-launch metrics out of `ncu --page raw --csv` exports (one line per launch)."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB", None), ("dram__bytes_write.sum", "MB", None),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1.0),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1.0),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1.0),
        ("launch__registers_per_thread", "regs", 1.0), ("launch__grid_size", "grid", 1.0)]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        print(path, "empty")
        continue
    h, units = rows[0], rows[1]
    col = {c: i for i, c in enumerate(h)}
    print(f"== {path}")
    for r in rows[2:]:
        name = r[col["Kernel Name"]][:48] if "Kernel Name" in col else "?"
        parts = []
        for k, label, scale in KEYS:
            if k not in col:
                continue
            v = float(r[col[k]].replace(",", "") or 0)
            u = units[col[k]]
            if label == "us":
                v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1e-3)
            elif label == "MB":
                v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
            parts.append(f"{label}={v:.1f}")
        print(f"  {name:48s} " + " ".join(parts))
