#!/bin/bash
# compose/decide occupancy A/B (DREG_COMPOSE_MINB 3 vs 4), two alternating rounds
for R in 1 2; do for MB in 3 4; do
  echo "MINB=$MB $(DREG_COMPOSE_MINB=$MB timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu --pairs-per-gpu 128 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value %.2f ms_per_step %.1f" % (d["value"], d["ms_per_step"]))')"
done; done
