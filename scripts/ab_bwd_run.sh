#!/bin/bash
# A/B of compositor-backward build variants under ab/ (see scripts/ab_build.sh):
# gradient agreement, the GPU test suite on the last variant, bench and
# per-kernel durations.
mkdir -p gpurun_out
vars="${VARS:-mg wz mgwz}"
for v in $vars; do
  python scripts/ab_bitwise.py base ab/$v/libvsx_b200.so > gpurun_out/abw_$v.log 2>&1
done
last="${vars##* }"
VSX_LIB=ab/$last/libvsx_b200.so python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$last.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/gpu_tests_$last.log
for v in base $vars base; do
  VSX_LIB=ab/$v/libvsx_b200.so python bench.py --cpu-tiles 0 > gpurun_out/bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_$v.log').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['ms_per_launch'],4))" >> gpurun_out/ab_summary.log 2>&1
done
for v in base $vars; do
  VSX_LIB=ab/$v/libvsx_b200.so bash scripts/kernel_times.sh raster_bwd 40 > gpurun_out/kt_$v.log 2>&1
  echo "$v $(cat gpurun_out/kt_$v.log)" >> gpurun_out/ab_summary.log
done
tail -n 2 gpurun_out/abw_*.log gpurun_out/gpu_tests_$last.log; cat gpurun_out/ab_summary.log
