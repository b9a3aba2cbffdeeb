#!/bin/bash
# Spectral-state kernel variants: plane (CTAs/SM x load batch) and x-pass (one-tile vs pipelined).
O=gpurun_out/ss3; mkdir -p $O
for V in "DREG_SS=1" "DREG_PLANE_SS=308" "DREG_PLANE_SS=204" "DREG_PLANE_SS=208" "DREG_PLANE_SS=216" "DREG_PIPE_SS=3" "DREG_PIPE_SS=4" "DREG_PIPE_SS=34" "DREG_PIPE_SS=44"; do
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
