#!/bin/bash
# Round-2 GPU check: pytest -m gpu, smoke, bench (config 3), reference arm, the
# single-pair config lines (1, 2, 4, 5) and the ncu launch list of one config-3 step.
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for C in 1 2 4 5; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 5 > $O/bench_config$C.json 2> $O/bench_config$C.err
done
if [ "${NCU:-1}" = 1 ]; then
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --pairs 32"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
fi
