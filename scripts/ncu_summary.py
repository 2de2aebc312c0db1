#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: a launch list (CSV) or a --set full report.

  python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
  python scripts/ncu_summary.py report gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>_ncu.txt
"""
import collections
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis",
            "Memory Workload Analysis", "Occupancy", "Launch Statistics",
            "Scheduler Statistics", "Warp State Statistics")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "launch__registers_per_thread")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        tot[name] += us
        cnt[name] += 1
    s = sum(tot.values())
    print(f"# ncu launch list ({sum(cnt.values())} launches, {s / 1e3:.3f} ms total, "
          "cold-cache serialised: compare shares)")
    print(f"{'total_ms':>10} {'share':>6} {'n':>5} {'avg_us':>9}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / 1e3:10.3f} {100 * v / s:5.1f}% {cnt[k]:5d} {v / cnt[k]:9.1f}  {k}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    si, mi, ui, vi = (h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"),
                      h.index("Metric Value"))
    kname = h.index("Kernel Name")
    print(f"# ncu --set full: {r[1][kname].split('(')[0]}")
    for row in r[1:]:
        if row[si] in SECTIONS and row[mi]:
            print(f"{row[si][:28]:28} | {row[mi]:45} | {row[vi]} {row[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hdr, units, vals = rr[0], rr[1], rr[2]
        print("# raw")
        for m in RAW:
            if m in hdr:
                j = hdr.index(m)
                print(f"{m:60} {vals[j]} {units[j]}")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
