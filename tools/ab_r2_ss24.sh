#!/bin/bash
O=gpurun_out/ss24; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=1240444" "DREG_PIPE_SS=1120434"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
