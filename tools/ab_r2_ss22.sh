#!/bin/bash
O=gpurun_out/ss22; mkdir -p $O
for V in "DREG_PIPE_SS=1120444" "DREG_PIPE_SS=1120448" "DREG_PIPE_SS=1120644" "DREG_PIPE_SS=1120248" "DREG_PIPE_SS=1160444" "DREG_PIPE_SS=1120424"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
