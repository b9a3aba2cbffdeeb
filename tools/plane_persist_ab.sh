#!/bin/bash
# Persistent plane pass (DREG_PLANE_PERSIST) vs per-plane CTAs: bit-identity and speed
for P in 0 1; do echo "PERSIST=$P $(DREG_PLANE_PERSIST=$P timeout 300 python tools/phi_digest.py 8 2>&1 | tail -1)"; done
for R in 1 2; do for P in 0 1; do
  echo "PERSIST=$P $(DREG_PLANE_PERSIST=$P timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("value %.2f plane_ms %.4f xpass_ms %.4f" % (d["value"], r["plane_ms"], r["xpass_ms"]))')"
done; done
