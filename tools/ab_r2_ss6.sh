#!/bin/bash
O=gpurun_out/ss6; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=120841" "DREG_PIPE_SS=120842" "DREG_PIPE_SS=120642" "DREG_PIPE_SS=160442" "DREG_PIPE_SS=120444"; do
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spectral or pipelined" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
