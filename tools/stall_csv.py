"""Read an ncu --csv --page raw dump on stdin; print warp-stall ratios and instruction totals."""
import csv
import sys

rows = [r for r in csv.reader(sys.stdin) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, v = rows[hdr], rows[hdr + 2]
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
        try:
            x = float(v[i])
        except ValueError:
            continue
        if x > 0.1:
            print(f"  stall {k[34:-23]:22s} {x:.2f}")
    if k in ("smsp__inst_executed.sum", "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"):
        print(f"  {k} {v[i]}")
