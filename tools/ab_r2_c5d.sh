#!/bin/bash
O=gpurun_out/c5d; mkdir -p $O
for V in "DREG_PLANE_PF=0" "DREG_PLANE_PF=1"; do
  env ${V//,/ } timeout 600 python bench.py --config 5 --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 > $O/bench_$V.json 2> $O/bench_$V.err
done
