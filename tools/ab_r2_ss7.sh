#!/bin/bash
O=gpurun_out/ss7; mkdir -p $O
for V in "DREG_SS=1" "DREG_PLANE_UPF=0" "DREG_PLANE_PF=0" "DREG_PLANE_PF=0,DREG_PLANE_UPF=0" "DREG_PLANE_PF=2"; do
  env ${V//,/ } timeout 600 python bench.py --no-cpu --no-e2e --allow-env --steps 2 --warmup 3 --pairs ${PAIRS:-128} > $O/bench_$V.json 2> $O/bench_$V.err
done
python tools/phi_digest.py 8 > $O/digest.txt 2>&1
