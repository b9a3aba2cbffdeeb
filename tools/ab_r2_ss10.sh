#!/bin/bash
O=gpurun_out/ss10; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=1120842" "DREG_PIPE_SS=1121241" "DREG_PIPE_SS=1120641" "DREG_PIPE_SS=1160841" "DREG_PIPE_SS=120442"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_guard.py -m gpu -x -q -k "spectral or pipelined or config3 or config2 or guard or schedule" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
