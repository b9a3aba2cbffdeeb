#!/bin/bash
# ncu --set full of the spectral-state kernels (PAIRS pairs per launch); the reports stay on
# the box, their raw / source pages come back as CSV.
O=gpurun_out/ncu_ss; mkdir -p $O
P=${PAIRS:-32}
CMD="python tools/profile_step.py $P 1"
$CMD > $O/plain.log 2>&1 || exit 1
for K in ${KERNELS:-xpass_pipe plane_reg}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o /tmp/$K env DREG_CHUNK=$P $CMD > $O/ncu_$K.log 2>&1
  ncu -i /tmp/$K.ncu-rep --page raw --csv > $O/${K}_raw.csv 2>&1
  ncu -i /tmp/$K.ncu-rep --page source --csv --print-source sass > $O/${K}_sass.csv 2>&1
  ncu -i /tmp/$K.ncu-rep --page details > $O/${K}_details.txt 2>&1
done
