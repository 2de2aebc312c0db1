#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over smoke()
# and a slice of the GPU parity tests, restricted to this library's kernels
# (kernel names containing "vsx"). Logs in gpurun_out/sanitize_*.log.
#   bash scripts/sanitize.sh
mkdir -p gpurun_out
F=(--kernel-name kns=vsx --print-limit 20 --error-exitcode 9)
SMOKE='import __graft_entry__ as g; g.smoke()'
K="train_steps_match_oracle_and_reference or render_gaussians or bin_lists_bitexact_vs or raster_forward or decoder_backward"
for tool in memcheck racecheck synccheck initcheck; do
  compute-sanitizer --tool $tool "${F[@]}" python -c "$SMOKE" > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?" | tee -a gpurun_out/sanitize_summary.txt
done
for tool in memcheck racecheck; do
  compute-sanitizer --tool $tool "${F[@]}" python -m pytest tests/test_gpu_parity.py -q -x -k "$K" \
    > gpurun_out/sanitize_${tool}_tests.log 2>&1
  echo "$tool tests rc=$?" | tee -a gpurun_out/sanitize_summary.txt
done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/sanitize_*.log | sort | uniq -c
