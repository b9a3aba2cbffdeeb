#!/bin/bash
O=gpurun_out/ss20; mkdir -p $O
timeout 200 python tools/phi_digest.py 4 > $O/digest.txt 2>&1 || echo "hung/failed" >> $O/digest.txt
timeout 200 env DREG_PIPE_SS=41120841 python tools/phi_digest.py 4 > $O/digest_nb4.txt 2>&1 || echo "hung/failed" >> $O/digest_nb4.txt
timeout 200 env DREG_SS_CHG=1 python tools/phi_digest.py 4 > $O/digest_chg.txt 2>&1 || echo "hung/failed" >> $O/digest_chg.txt
for V in "DREG_SS=1" "DREG_PIPE_SS=41120841" "DREG_PIPE_SS=1240841"; do
  env ${V//,/ } timeout 300 python bench.py --no-cpu --no-e2e --allow-env --steps 3 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
