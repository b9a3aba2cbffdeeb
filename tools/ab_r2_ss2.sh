#!/bin/bash
# Spectral-state kernel timings: bench (64 pairs) across x-pass warp splits.
O=gpurun_out/ss2; mkdir -p $O
for V in "DREG_SS=0" "DREG_SS_CHG=1" "DREG_SS=1" "DREG_PIPE_SS=40841" "DREG_PIPE_SS=80441" "DREG_PIPE_SS=80442" "DREG_PIPE_SS=40841,DREG_SS_CHG=1"; do
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
