#!/bin/bash
# Spectral-state x-pass: warp splits (12 FFT warps) and packed-arithmetic library variants.
O=gpurun_out/ss4; mkdir -p $O
VD=paper_2109_12688_b200/lib/variants
for V in "DREG_SS=1" "DREG_PIPE_SS=120441" "DREG_PIPE_SS=120442" "DREG_PIPE_SS=120422" "DREG_LIB=$VD/libdreg_cuda_x1.so" "DREG_LIB=$VD/libdreg_cuda_x2.so" "DREG_LIB=$VD/libdreg_cuda_x1.so,DREG_PIPE_SS=120441" "DREG_LIB=$VD/libdreg_cuda_x2.so,DREG_PIPE_SS=120441"; do
  N=$(echo $V | tr '/' '_')
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$N.json 2> $O/bench_$N.err
done
python tools/phi_digest.py 8 > $O/digest.txt 2>&1
