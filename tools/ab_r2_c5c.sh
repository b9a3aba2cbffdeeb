#!/bin/bash
O=gpurun_out/c5c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "config5 or cluster" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for V in "DREG_CLUSTER=0" "DREG_CLUSTER=1" "DREG_CLUSTER=2"; do
  env ${V//,/ } timeout 600 python bench.py --config 5 --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 > $O/bench_$V.json 2> $O/bench_$V.err
done
