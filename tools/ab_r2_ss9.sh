#!/bin/bash
O=gpurun_out/ss9; mkdir -p $O
timeout 120 env DREG_PIPE_SS=1120442 python tools/phi_digest.py 4 > $O/digest_split.txt 2>&1 || { echo "split variant failed/hung" >> $O/digest_split.txt; exit 0; }
python tools/phi_digest.py 4 > $O/digest_base.txt 2>&1
for V in "DREG_SS=1" "DREG_PIPE_SS=1120442" "DREG_PIPE_SS=1120841" "DREG_PIPE_SS=1160442" "DREG_PIPE_SS=1240442"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
timeout 300 env DREG_PIPE_SS=1120442 DREG_SS_CHG=1 python tools/phi_digest.py 4 > $O/digest_split_chg.txt 2>&1
