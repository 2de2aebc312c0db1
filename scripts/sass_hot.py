#!/usr/bin/env python
"""Per-instruction stall samples of one kernel from an ncu source page (SASS).

  ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
  python scripts/sass_hot.py sass.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, ismp, iex = (h.index("Address"), h.index("Source"),
                       h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"))
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_")]
recs = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # only the first kernel of a multi-kernel page
    if len(r) <= iex:
        continue
    smp = float(r[ismp] or 0)
    ex = float(r[iex] or 0)
    st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    recs.append((r[ia], r[isrc], smp, ex, st))
tot = sum(x[2] for x in recs) or 1
totx = sum(x[3] for x in recs) or 1
print(f"# samples {tot:.0f}, warp instructions {totx:.4g}")
mode = sys.argv[2] if len(sys.argv) > 2 else "all"
for a, s, smp, ex, st in recs:
    if mode == "all" or smp / tot > float(mode):
        tops = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
        print(f"{a:>6} {100 * smp / tot:5.2f}% {ex / totx * 100:5.2f}%x  {s[:60]:60s} {tops}")

if mode == "regions":
    pass
