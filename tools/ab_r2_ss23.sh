#!/bin/bash
O=gpurun_out/ss23; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_guard.py -m gpu -x -q -k "spectral or pipelined or config3 or config2 or guard or schedule or config1 or identity" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for V in "DREG_PIPE256=1" "DREG_PIPE256=2"; do
  env ${V//,/ } timeout 600 python bench.py --config 5 --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 > $O/bench_c5_$V.json 2> $O/bench_c5_$V.err
done
for V in "DREG_SS=0" "DREG_SS=0,DREG_PIPE=40842"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs 128 > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 600 python bench.py --no-cpu > $O/bench256.json 2> $O/bench256.err
