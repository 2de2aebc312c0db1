#!/usr/bin/env python
"""Issue-stall breakdown (share of smsp__average_warps_issue_stalled_*) of an ncu report.

  python scripts/ncu_stalls.py rep.ncu-rep >> profiles/rNN_<kernel>_ncu.txt
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
items = []
for k in h:
    if k.startswith(pre) and k.endswith(suf):
        try:
            items.append((float(d[k].replace(",", "")), k[len(pre):-len(suf)]))
        except ValueError:
            pass
tot = sum(x for x, _ in items) or 1.0
print("# issue-stall reasons (share of stalled warp-cycles per issued instruction)")
for val, k in sorted(items, reverse=True)[:10]:
    print(f"stall {k:28s} {val:6.2f} {100 * val / tot:5.1f}%")
for k in ("smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"):
    print(k, d.get(k))
