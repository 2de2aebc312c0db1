#!/bin/bash
# usage: scripts/kernel_times.sh REGEX [count] -- per-kernel ncu durations over
# a short bench run (cold-cache, serialised: compare kernels, not steps).
re="$1"; cnt="${2:-60}"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$re" -c "$cnt" --csv \
  python bench.py --steps 2 --warmup 3 --cpu-tiles 0 > gpurun_out/kt.csv 2>/dev/null
python - <<'PY'
import csv, collections
d = collections.defaultdict(list)
for r in csv.reader(open("gpurun_out/kt.csv")):
    if len(r) > 10 and r[12] == "gpu__time_duration.sum":
        d[r[4].split("(")[0]].append(float(r[-1].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:44s} n={len(v):4d} mean_us={sum(v)/len(v)/1e3:9.1f} share={sum(v)/tot*100:5.1f}%")
PY
