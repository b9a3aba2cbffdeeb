#!/bin/bash
# plane_reg_kernel L2-prefetch distance sweep (DREG_PLANE_PF, in CTAs; resident wave = 148 x 3)
for PF in 1 0 74 148 296 444 888; do
  echo "PF=$PF $(DREG_PLANE_PF=$PF timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --pairs-per-gpu 64 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("value %.2f plane_ms %.4f xpass_ms %.4f" % (d["value"], r["plane_ms"], r["xpass_ms"]))')"
done
