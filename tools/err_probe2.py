"""Per-application w_update error (GPU fp32 FFT vs oracle fp64) and a 200-iteration solve."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from conftest import max_abs, random_field, rel_l2  # noqa: E402
from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, dreg, synth  # noqa: E402

o = CpuLib("oracle")
ctx = dreg.Context(0)
for shape in [(64, 64, 64), (32, 64, 128), (64, 128, 128)]:
    v, b = random_field(shape, 5, 1.0), random_field(shape, 6, 1.0)
    for (n, lam, th) in [(3, 0.05, 0.5), (2, 0.1, 1.0), (1, 2.0, 0.1)]:
        cfg = abi.solver_cfg(order=n, lambda_=lam, theta=th)
        g, r = ctx.w_update(v, b, cfg), o.w_update(v, b, cfg)
        print(shape, n, f"w rel-L2 {rel_l2(g, r):.2e} max-abs/max {max_abs(g, r) / np.abs(r).max():.2e}")
f, m = synth.make_pair(4, 4, (64, 64, 64))
for iters in (20, 50, 200):
    s = abi.solver_cfg(data_term=2, order=3, lambda_=0.05, theta=0.5, max_iters=iters, log_objective=False)
    v1, d1 = ctx.solve_velocity(f, m, s)
    v2, d2 = o.solve_velocity(f, m, s)
    print("solve", iters, f"v rel-L2 {rel_l2(v1, v2):.2e} max-abs {max_abs(v1, v2):.2e}  |v|max {np.abs(v2).max():.3f}")
