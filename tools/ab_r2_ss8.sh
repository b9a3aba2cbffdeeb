#!/bin/bash
O=gpurun_out/ss8; mkdir -p $O
for V in "DREG_SS=1" "DREG_PIPE_SS=2060242" "DREG_PIPE_SS=2060244" "DREG_PIPE_SS=2060442" "DREG_PIPE_SS=2040442"; do
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
DREG_PIPE_SS=2060242 python tools/phi_digest.py 8 > $O/digest.txt 2>&1
python tools/phi_digest.py 8 >> $O/digest.txt 2>&1
