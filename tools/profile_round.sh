#!/bin/bash
# Round evidence on the GPU box: bench line, reference arm, ncu launch list of one bench
# step and --set full captures of the per-iteration kernels, summarised into
# gpurun_out/prof/ (copied to profiles/ by hand).   tools/profile_round.sh <tag>
TAG=${1:-r1c}
O=gpurun_out; mkdir -p $O/prof
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --pairs-per-gpu 32"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
R=""
for K in xpass_pipe plane_reg compose_decide; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o /tmp/$K python tools/profile_step.py 32 1 > $O/ncu_$K.log 2>&1
  ncu -i /tmp/$K.ncu-rep --page source --csv --print-source sass > $O/${K}_sass.csv 2>&1
  R="$R,/tmp/$K.ncu-rep"
done
DREG_PROF_DIR=$O/prof python tools/ncu_summary.py $TAG $O/launches.csv ${R#,} 32 "$CMD" > $O/summary.log 2>&1
