#!/bin/bash
# Cost of L2-prefetching planes of finished pairs (DREG_PLANE_PF=-1: unconditional, the old behaviour)
O=gpurun_out/dead; mkdir -p $O
for r in 1 2; do for V in "DREG_PLANE_PF=-1" "DREG_PLANE_PF=1"; do
  env $V timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 > $O/bench_${V}_r$r.json 2> $O/bench_${V}_r$r.err
done; done
