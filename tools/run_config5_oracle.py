"""Full-size config 4 on the CPU oracle (256x256x192, n=2, 10 fields x 50 iterations):
folding count / min det J / phi digests into tests/golden/config5_oracle.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, synth  # noqa: E402

c = synth.CONFIGS["config5"]
f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
t0 = time.time()
o = CpuLib("oracle")
phi, warped, res = o.register_pair(f, m, synth.config_cfg("config5"))
js = o.jacobian_stats(phi)
lg = abi.level_logs(res)[0]
np.save("/tmp/config5_oracle_phi.npy", phi)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "config5_phi_sub8.npz"), phi=phi[::8, ::8, ::8].copy())
json.dump({"config": "config5", "velocity_count": res.velocity_count, "solves": res.solves,
           "mean_sad": lg["mean_sad"], "folding": int(js.nonpositive), "min_det": js.min_det,
           "phi_sum": float(phi.astype(np.float64).sum()), "phi_sumsq": float((phi.astype(np.float64) ** 2).sum()),
           "seconds": time.time() - t0}, open(os.path.join(ROOT, "tests", "golden", "config5_oracle.json"), "w"), indent=1)
print("done", res.velocity_count, js.nonpositive, time.time() - t0)
