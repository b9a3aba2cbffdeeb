#!/bin/bash
# Which part of the spectral-state x-pass sets its rate?  An experiments build (make EXPERIMENTS=1,
# copied to lib/variants/libdreg_cuda_exp.so) can skip parts of the kernel in the timing loop only
# (DREG_DBG_SKIP_TK: 1 = the x-FFT arithmetic, 2 = the point-wise stage, 4 = the spectrum staging loads).
O=gpurun_out/skip; mkdir -p $O; rm -f $O/skip.txt
L=paper_2109_12688_b200/lib/variants/libdreg_cuda_exp.so
for S in 0 1 2 4 3 5 6 7; do
  echo "skip=$S $(DREG_LIB=$L DREG_DBG_SKIP_TK=$S DREG_CHUNK=128 timeout 300 python tools/profile_step.py 128 1 2>&1 | head -1)" >> $O/skip.txt
done
