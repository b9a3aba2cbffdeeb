#!/bin/bash
# compute-sanitizer over the registration path: memcheck, racecheck,
# synccheck, initcheck on tools/sanitize_run.py at three grids.  Logs go to
# gpurun_out/sanitizer/<tool>_<grid>.txt; a summary line per run to summary.txt.
# Usage (GPU box): bash tools/sanitize.sh [tools...]
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitizer
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
TOOLS=${*:-memcheck racecheck synccheck initcheck}
# grid (z,y,x) : what it covers
#  16,32,32   generic x-pass (M = 32) + plane_fast_kernel
#  64,64,64   xpass_fast (R2 = 4) + xpass_pipe (M = 64) + plane_reg <64,64>
#  64,128,128 the bench grid: xpass_fast/pipe (M = 128) + plane_reg <128,64>
GRIDS="16,32,32 64,64,64 64,128,128"
for tool in $TOOLS; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  [ "$tool" = memcheck ] && extra="--leak-check full"
  for g in $GRIDS; do
    tag="${tool}_${g//,/x}"
    args="--shape $g --pairs 2 --warps 2 --iters 4"
    [ "$g" = "16,32,32" ] && args="$args --data-term 1"
    start=$(date +%s)
    timeout 900 $CS --tool "$tool" $extra --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_run.py $args > "$OUT/$tag.txt" 2>&1
    rc=$?
    echo "$tag rc=$rc $(( $(date +%s) - start ))s :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' "$OUT/$tag.txt" | tr '\n' ' ')" | tee -a "$OUT/summary.txt"
  done
done
# precise-mode (fp64 FFT) x-pass / split plane path once under memcheck + racecheck
for tool in memcheck racecheck; do
  tag="${tool}_precise_64x64x64"
  timeout 900 $CS --tool "$tool" --error-exitcode 99 --print-limit 50 \
    python tools/sanitize_run.py --shape 64,64,64 --pairs 2 --warps 1 --iters 3 --precise 1 > "$OUT/$tag.txt" 2>&1
  echo "$tag rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$OUT/$tag.txt" | tr '\n' ' ')" | tee -a "$OUT/summary.txt"
done
