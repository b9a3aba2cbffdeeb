#!/bin/bash
O=gpurun_out/c4; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_cufft_xcheck.py -m gpu -x -q -s -k "config4 or precise or cluster or config5 or cufft" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for V in "DREG_CLUSTER=0" "DREG_CLUSTER=1"; do
  env ${V//,/ } timeout 600 python bench.py --config 4 --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 > $O/bench_$V.json 2> $O/bench_$V.err
done
