#!/bin/bash
O=gpurun_out/ss16; mkdir -p $O
for V in "DREG_SS=1" "DREG_XPASS_SMS=132" "DREG_XPASS_SMS=116" "DREG_XPASS_SMS=100"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
