import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2109_12688_b200 import abi, dreg, synth
from oracle.oracle import CpuLib
o = CpuLib("oracle")
F, M = synth.make_batch(1, 300, 3, (16, 32, 32))
s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=30, log_objective=False)
cfg = abi.reg_cfg(s, 1, (4,), (30,))
po, wo, ro = o.register_pair(F[0], M[0], cfg)
print("oracle sad", abi.level_logs(ro)[0]['mean_sad'][:2])
mode = sys.argv[1]
ctx = dreg.Context(0)
if mode == "single_first":
    p1, w1, r1 = ctx.register_pair(F[0], M[0], cfg); print("single", abi.level_logs(r1)[0]['mean_sad'][:2], np.abs(p1-po).max())
    phis, warps, res = ctx.register_batch(list(F), list(M), cfg); print("batch", abi.level_logs(res[0])[0]['mean_sad'][:2], np.abs(phis[0]-po).max())
    p1, w1, r1 = ctx.register_pair(F[0], M[0], cfg); print("single", abi.level_logs(r1)[0]['mean_sad'][:2], np.abs(p1-po).max())
else:
    phis, warps, res = ctx.register_batch([F[0]]*3, [M[0]]*3, cfg); print("batch same", [abi.level_logs(r)[0]['mean_sad'][:2] for r in res], [np.abs(p-po).max() for p in phis])
    phis, warps, res = ctx.register_batch([F[0]], [M[0]], cfg); print("batch1", [abi.level_logs(r)[0]['mean_sad'][:2] for r in res], [np.abs(p-po).max() for p in phis])
