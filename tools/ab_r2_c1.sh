#!/bin/bash
O=gpurun_out/c1; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_reference_pins.py -m gpu -x -q -k "not slow" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for V in "DREG_SS=0" "DREG_SS=1"; do
  env ${V//,/ } timeout 600 python bench.py --config 1 --no-cpu --allow-env --steps 30 --warmup 5 > $O/bench_c1_$V.json 2> $O/bench_c1_$V.err
done
timeout 600 python bench.py --config 2 --no-cpu --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
