#!/bin/bash
O=gpurun_out/ss19; mkdir -p $O
python tools/phi_digest.py 4 > $O/digest.txt 2>&1
DREG_SS_CHG=1 python tools/phi_digest.py 4 > $O/digest_chg.txt 2>&1
DREG_SS=0 python tools/phi_digest.py 4 > $O/digest_ss0.txt 2>&1
for V in "DREG_SS=1" "DREG_SS=0" "DREG_PIPE_SS=120442" "DREG_PIPE_SS=41120841"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
