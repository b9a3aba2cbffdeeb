#!/bin/bash
# Round evidence on the GPU box: bench line, reference arm, ncu launch list of one bench
# step and --set full captures of the per-iteration kernels, summarised into
# gpurun_out/prof/ (copied to profiles/ by hand).   tools/profile_round.sh <tag>
TAG=${1:-r1c}
P=${PAIRS:-32}   # pairs per launch for the launch list and the full captures
O=gpurun_out; mkdir -p $O/prof
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --pairs-per-gpu $P"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
R=""
for K in xpass_pipe plane_reg compose_decide; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o /tmp/$K env DREG_CHUNK=$P python tools/profile_step.py $P 1 > $O/ncu_$K.log 2>&1
  ncu -i /tmp/$K.ncu-rep --page source --csv --print-source sass > $O/${K}_sass.csv 2>&1
  R="$R,/tmp/$K.ncu-rep"
done
DREG_PROF_DIR=$O/prof python tools/ncu_summary.py $TAG $O/launches.csv ${R#,} $P "$CMD" > $O/summary.log 2>&1
# plane prefetch distance (waves of resident CTAs) 1 vs 2 vs 3
for PF in 1 2 3; do
  echo "PF=$PF $(DREG_PLANE_PF=$PF timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --pairs-per-gpu 128 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("value %.2f plane_ms %.4f xpass_ms %.4f" % (d["value"], r["plane_ms"], r["xpass_ms"]))')" >> $O/pf2.log
done
