#!/bin/bash
O=gpurun_out/ss12; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=1120861" "DREG_PLANE_STREAM=0"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
python tools/phi_digest.py 4 > $O/digest.txt 2>&1
timeout 600 python bench.py --no-cpu > $O/bench256.json 2> $O/bench256.err
