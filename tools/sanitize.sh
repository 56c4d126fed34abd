#!/bin/bash
# compute-sanitizer sweep over the product kernels (run on the GPU box):
#   bash tools/sanitize.sh [OUTDIR]
# memcheck / racecheck / synccheck / initcheck on one C1 and one C2 estimate_maps
# (tools/one_step.py), every kernel in the process (ours and the cuBLAS/cuSOLVER ones).
set -u
OUT=${1:-gpurun_out/sanitizer}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in C1 C2; do
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
    echo "== $cfg $tool" | tee -a "$OUT/summary.txt"
    timeout 900 $CS --tool $tool $extra --print-limit 50 --error-exitcode 99 \
      python tools/one_step.py $cfg 2 > "$OUT/${cfg}_${tool}.log" 2>&1
    rc=$?
    echo "rc=$rc" | tee -a "$OUT/summary.txt"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|Error|hazard" "$OUT/${cfg}_${tool}.log" | tail -5 | tee -a "$OUT/summary.txt"
  done
done
