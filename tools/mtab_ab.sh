#!/bin/bash
# (experiment record: the DREG_MTAB knob exists only with profiles/r1j_mtab.patch applied)
# plane multiplier table (DREG_MTAB=1, default) vs the inline power + reciprocal (DREG_MTAB=0):
# bit-identity of phi and speed.  Output under gpurun_out/.
O=gpurun_out; mkdir -p $O
for X in 0 1; do echo "MTAB=$X $(DREG_MTAB=$X timeout 300 python tools/phi_digest.py 8 2>&1 | tail -1)"; done
for R in 1 2; do for X in 0 1; do
  echo "MTAB=$X $(DREG_MTAB=$X timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("value %.2f xpass_ms %.4f plane_ms %.4f frac %.4f iter_frac %.4f steps %s" % (d["value"], r["xpass_ms"], r["plane_ms"], r["frac"], r["iteration_frac"], d.get("step_ms_rank0")))')"
done; done
