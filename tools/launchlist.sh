#!/bin/bash
O=gpurun_out; mkdir -p $O
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --pairs ${PAIRS:-64}"
$CMD > $O/ll_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
