"""Config 4 (128^3 swirl, n = 3, 15 fields x 200 iterations) on the CPU oracle, phi
stored on the [::2]^3 sub-grid (tests/golden/config4_phi_sub2.phi.xz, 2^-16 voxel
quantisation, tools/run_config3_phi.save) and checked against the recorded digest in
tests/golden/config4_oracle.json.  ~25 CPU-minutes.

    python tools/run_config4_phi.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import synth  # noqa: E402
from run_config3_phi import save  # noqa: E402

c = synth.CONFIGS["config4"]
f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
t0 = time.time()
phi, _, res = CpuLib("oracle").register_pair(f, m, synth.config_cfg("config4"))
rec = json.load(open(os.path.join(ROOT, "tests", "golden", "config4_oracle.json")))
assert res.velocity_count == rec["velocity_count"]
assert float(phi.astype(np.float64).sum()) == rec["phi_sum"], "oracle run differs from the recorded digest"
save(os.path.join(ROOT, "tests", "golden", "config4_phi_sub2.phi.xz"), phi[::2, ::2, ::2].copy())
print("done", res.velocity_count, time.time() - t0)
