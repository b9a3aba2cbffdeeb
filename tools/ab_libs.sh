#!/bin/bash
# A/B kernel timing across library variants: tools/ab_libs.sh <pairs> lib1.so lib2.so ...
# (default library first), each via tools/profile_step.py (per-kernel CUDA-event loop).
P=$1; shift
echo "default: $(python tools/profile_step.py $P 1 | head -1)"
for L in "$@"; do echo "$L: $(DREG_LIB=$L python tools/profile_step.py $P 1 | head -1)"; done
echo "default again: $(python tools/profile_step.py $P 1 | head -1)"
