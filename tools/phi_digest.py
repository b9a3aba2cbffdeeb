"""Register a small config-2 batch and print a digest of phi (compare kernel variants
selected by DREG_* env knobs for bit-identity):  python tools/phi_digest.py [pairs]"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2109_12688_b200 import dreg, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
F, M = synth.make_batch(3, 1000, B, (64, 128, 128))
cfg = synth.config_cfg("config3")
with dreg.Context(0) as ctx:
    phis, warps, res = ctx.register_batch(list(F), list(M), cfg, want_warped=False)
h = hashlib.sha256()
for p in phis:
    h.update(np.ascontiguousarray(p).tobytes())
print("digest", h.hexdigest()[:16], "velocity", [r.velocity_count for r in res], "solves", [r.solves for r in res],
      "sum", float(sum(np.abs(p).astype(np.float64).sum() for p in phis)))
