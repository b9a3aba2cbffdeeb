#!/bin/bash
O=gpurun_out/ss14; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_cufft_xcheck.py tests/test_golden.py -m gpu -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for V in "DREG_SS=1"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
