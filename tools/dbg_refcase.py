"""Debug: GPU vs oracle on the reference's synthetic cases under config variants."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, dreg  # noqa: E402

ref, ora = CpuLib("reference"), CpuLib("oracle")
ctx = dreg.Context(0)


def cmp(tag, t, s, cfg, prec=0):
    ctx.set_precision(prec)
    phi, w, res = ctx.register_pair(t, s, cfg)
    po, wo, ro = ora.register_pair(t, s, cfg)
    err = np.abs(phi.astype(np.float64) - po).max()
    rel = np.linalg.norm(phi.astype(np.float64) - po) / max(np.linalg.norm(po), 1e-30)
    lv = [(res.per_level[l].warps, ro.per_level[l].warps) for l in range(res.levels)]
    its = [[res.per_level[l].solver_iterations[i] for i in range(res.per_level[l].warps)] for l in range(res.levels)]
    itso = [[ro.per_level[l].solver_iterations[i] for i in range(ro.per_level[l].warps)] for l in range(ro.levels)]
    sad = [[round(res.per_level[l].mean_sad[i], 7) for i in range(res.per_level[l].warps + 1)] for l in range(res.levels)]
    sado = [[round(ro.per_level[l].mean_sad[i], 7) for i in range(ro.per_level[l].warps + 1)] for l in range(ro.levels)]
    print(f"{tag}: err {err:.3e} rel {rel:.3e} vc {res.velocity_count}/{ro.velocity_count} warps {lv}")
    if its != itso:
        print("   iters", its, itso)
    print("   sad gpu", sad)
    print("   sad ora", sado)


t, s, tl, sl = ref.make_case("sphere_ellipsoid", (32, 32, 32))
for dt in (1, 2):
    for lv in (1, 2, 3):
        sol = abi.solver_cfg(data_term=dt, order=2, lambda_=10.0, theta=0.05, log_objective=False)
        cfg = dreg.make_registration_config(abi.DREG_PROFILE_CAPPED, sol, lv)
        cmp(f"dt{dt} levels{lv}", t, s, cfg)
sol = abi.solver_cfg(data_term=1, order=2, lambda_=10.0, theta=0.05, log_objective=False)
cfg = dreg.make_registration_config(abi.DREG_PROFILE_CAPPED, sol, 3)
cmp("dt1 levels3 precise", t, s, cfg, prec=2)
# single solve at 32^3
w, d = ctx.solve_velocity(t, s, sol)
wo, do = ora.solve_velocity(t, s, sol)
print("single solve dt1: err", np.abs(w - wo).max(), "rel", np.linalg.norm(w - wo) / np.linalg.norm(wo))
for n in (8, 16):
    a, b = t[::32 // n, ::32 // n, ::32 // n].copy(), s[::32 // n, ::32 // n, ::32 // n].copy()
    w, d = ctx.solve_velocity(a, b, sol)
    wo, do = ora.solve_velocity(a, b, sol)
    print(f"single solve {n}^3 dt1: err", np.abs(w - wo).max(), "rel", np.linalg.norm(w - wo) / np.linalg.norm(wo))
