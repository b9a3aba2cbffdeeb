#!/bin/bash
O=gpurun_out/ss13; mkdir -p $O
VD=paper_2109_12688_b200/lib/variants
for V in "DREG_SS=1" "DREG_LIB=$VD/libdreg_cuda_x1.so" "DREG_LIB=$VD/libdreg_cuda_x2.so"; do
  N=$(echo $V | tr '/' '_')
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$N.json 2> $O/bench_$N.err
done
KERNELS=xpass_pipe bash tools/ncu_ss.sh
