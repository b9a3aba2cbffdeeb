#!/bin/bash
# config 5: pipelined x-pass at M = 256 (two-buffer ring) vs one tile per CTA; parity test of the config-5 grid
O=gpurun_out/c5; mkdir -p $O
for V in "DREG_PIPE256=0" "DREG_PIPE256=1" "DREG_PIPE256=2"; do
  env ${V//,/ } timeout 600 python bench.py --config 5 --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config5" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
