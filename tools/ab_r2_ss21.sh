#!/bin/bash
O=gpurun_out/ss21; mkdir -p $O
python tools/phi_digest.py 4 > $O/digest.txt 2>&1
for V in "DREG_SS=1" "DREG_PIPE_SS=1120842" "DREG_PIPE_SS=1120844" "DREG_PIPE_SS=1120442"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
