#!/bin/bash
O=gpurun_out/c45; mkdir -p $O
for C in 5 4; do
for V in "DREG_SS=1" "DREG_PIPE256=2"; do
  [ $C = 4 ] && [ "$V" != "DREG_SS=1" ] && continue
  env ${V//,/ } timeout 600 python bench.py --config $C --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 > $O/bench_c${C}_$V.json 2> $O/bench_c${C}_$V.err
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config5 or config4 or split or precise" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
