#!/bin/bash
O=gpurun_out/ft; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "cluster or m256 or spectral or pipelined" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
