#!/bin/bash
# config 5: 2-CTA cluster plane kernel vs the 3-pass split; parity tests on the config-5 grid
O=gpurun_out/c5b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config5" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for V in "DREG_CLUSTER=0" "DREG_CLUSTER=1"; do
  env ${V//,/ } timeout 600 python bench.py --config 5 --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 > $O/bench_$V.json 2> $O/bench_$V.err
done
