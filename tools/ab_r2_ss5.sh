#!/bin/bash
# Spectral-state x-pass warp splits (after fast division + incremental staging), then the new tests.
O=gpurun_out/ss5; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=80842" "DREG_PIPE_SS=81241" "DREG_PIPE_SS=81221" "DREG_PIPE_SS=121241" "DREG_PIPE_SS=80851" "DREG_PIPE_SS=120442"; do
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spectral or pipelined or config3 or config2 or identity" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
