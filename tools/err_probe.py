"""Parity error of a long registration (config-4 settings on 64^3) under env knobs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from conftest import max_abs, rel_l2  # noqa: E402
from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, dreg, synth  # noqa: E402

warps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
f, m = synth.make_pair(4, 4, (64, 64, 64))
c = synth.CONFIGS["config4"]
s = abi.solver_cfg(data_term=2, order=3, lambda_=0.05, theta=0.5, max_iters=200, log_objective=False)
cfg = abi.reg_cfg(s, 1, (warps,), (200,))
cache = f"/tmp/oracle_c4_{warps}.npy"
if os.path.exists(cache):
    po = np.load(cache)
else:
    po, _, ro = CpuLib("oracle").register_pair(f, m, cfg)
    np.save(cache, po)
with dreg.Context(0) as ctx:
    p, w, r = ctx.register_pair(f, m, cfg)
print(os.environ.get("TAG", ""), f"warps {warps} max-abs {max_abs(p, po):.3e} rel-L2 {rel_l2(p, po):.3e} vc {r.velocity_count}")
