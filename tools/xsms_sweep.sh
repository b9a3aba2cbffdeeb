#!/bin/bash
# x-pass throughput vs persistent CTA count (DREG_XPASS_SMS): can it keep HBM saturated
# on a subset of the SMs (leaving the rest for a concurrent plane pass)?
for S in 148 136 124 112 100 88; do
  echo "SMS=$S $(DREG_XPASS_SMS=$S timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --pairs-per-gpu 64 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("value %.2f xpass_ms %.4f frac %.3f plane_ms %.4f" % (d["value"], r["xpass_ms"], r["frac"], r["plane_ms"]))')"
done
