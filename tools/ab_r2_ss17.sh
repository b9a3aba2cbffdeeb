#!/bin/bash
O=gpurun_out/ss17; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=1240841" "DREG_PIPE_SS=1240641" "DREG_PIPE_SS=1180841"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 300 env DREG_PIPE_SS=1240841 python tools/phi_digest.py 4 > $O/digest_24.txt 2>&1
python tools/phi_digest.py 4 > $O/digest.txt 2>&1
