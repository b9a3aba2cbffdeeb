#!/bin/bash
# Spectral-state iteration A/B: parity tests, then the bench with the real-space state
# (DREG_SS=0), the spectral state with the change norm (DREG_SS_CHG=1) and without it.
O=gpurun_out/ss; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
DREG_SS_CHG=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config2 or config3 or config_3 or config_2" > $O/tests_chg.log 2>&1; echo rc=$? >> $O/tests_chg.log
for V in "DREG_SS=0" "DREG_SS_CHG=1" "DREG_SS=1" $EXTRA; do
  env $V timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 > $O/bench_$V.json 2> $O/bench_$V.err
done
