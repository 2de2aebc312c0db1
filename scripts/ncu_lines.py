#!/usr/bin/env python
"""Per-CUDA-line instruction counts and stall samples of an ncu report
(captured with -lineinfo and --import-source on).

  python scripts/ncu_lines.py rep.ncu-rep [top] [file-substring]
Prints the top lines by warp-stall samples, then the totals per line range
named in RANGES (edit to the kernel's phases).
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
only = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines = []
fname = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))

    def num(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    lines.append((fname, int(r[0]), r[1].strip(), num("Warp Stall Sampling (All Samples)"),
                  num("Instructions Executed")))
if only:
    lines = [x for x in lines if only in (x[0] or "")]
ts = sum(x[3] for x in lines) or 1.0
ti = sum(x[4] for x in lines) or 1.0
print(f"# {len(lines)} lines, {ts:.0f} stall samples, {ti / 1e6:.1f} M warp instructions")
print(f"{'samp%':>6s} {'inst%':>6s} {'Minst':>7s}  file:line  source")
for f, ln, src, s, i in sorted(lines, key=lambda x: -x[3])[:top]:
    short = (f or "?").rsplit("/", 1)[-1]
    print(f"{100 * s / ts:6.2f} {100 * i / ti:6.2f} {i / 1e6:7.2f}  {short}:{ln}  {src[:90]}")

# optional phase ranges: VSX_RANGES="name:lo-hi,name:lo-hi" over the selected file's lines
import os  # noqa: E402
rs = os.environ.get("VSX_RANGES")
if rs:
    acc = {}
    for f, ln, src, s, i in lines:
        name = "other"
        for part in rs.split(","):
            nm, span = part.split(":")
            lo, hi = (int(x) for x in span.split("-"))
            if lo <= ln <= hi and (f or "").endswith(os.environ.get("VSX_RANGES_FILE", "")):
                name = nm
        a = acc.setdefault(name, [0.0, 0.0])
        a[0] += s
        a[1] += i
    for nm, (s, i) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        print(f"{nm:12s} samples {100 * s / ts:5.1f}%  instructions {100 * i / ti:5.1f}% ({i / 1e6:.1f} M)")
