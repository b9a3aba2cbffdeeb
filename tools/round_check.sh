#!/bin/bash
# Full GPU check: pytest -m gpu, smoke, bench (default), reference arm, and bench under
# torchrun with one process (the driver's N>1 launch path, NCCL init + all-gather).
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu > $O/bench_torchrun.json 2> $O/bench_torchrun.err
