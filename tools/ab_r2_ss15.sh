#!/bin/bash
O=gpurun_out/ss15; mkdir -p $O
timeout 300 python tools/phi_digest.py 4 > $O/digest.txt 2>&1
timeout 300 env DREG_SS_CHG=1 python tools/phi_digest.py 4 > $O/digest_chg.txt 2>&1
timeout 300 env DREG_PIPE_SS=3 python tools/phi_digest.py 4 > $O/digest_onetile.txt 2>&1
for V in "DREG_SS=1" "DREG_PIPE_SS=120442" "DREG_PIPE_SS=1120442" "DREG_SS_CHG=1"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spectral or config3 or config2 or pipelined" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
