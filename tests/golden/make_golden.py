"""Generate tests/golden/ref_fixtures.npz from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref/libdreg_ref.so, which is compiled from
/root/reference/proj/core/src by `make -C oracle ref`):

    python tests/golden/make_golden.py

The reference ships no golden vectors; every input here is seeded
std::mt19937 with gen()/2^32 like the reference tests (tests/oracles.hpp:19-27), and
every output is what dreg:: computed for it.  tests/test_golden.py checks the C
restatement (oracle/) bit-for-bit against these and the GPU path within tolerance.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from conftest import random_field, random_volume, smooth_random_field  # noqa: E402
from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, synth  # noqa: E402


def main():
    ref = CpuLib("reference")
    out = {}
    # spectral symbol (regularizer.cpp:51-79)
    for n, dims in [(1, (4, 6, 5)), (2, (8, 4, 6)), (3, (5, 5, 4))]:
        out[f"symbol_n{n}"] = ref.laplacian_symbol(n, dims)
    # point-wise v-updates (admm.cpp:23-63), 6^3
    shp = (6, 6, 6)
    t, w = random_volume(shp, 101), random_volume(shp, 102)
    g, wh, bh = random_field(shp, 103, 1.0), random_field(shp, 104, 1.0), random_field(shp, 105, 1.0)
    out.update(vu_target=t, vu_warped=w, vu_grad=g, vu_w_hat=wh, vu_b_hat=bh)
    for dt in (1, 2):
        out[f"vu_out_s{dt}"] = ref.v_update(t, w, g, wh, bh, abi.solver_cfg(data_term=dt, theta=0.07))
    # w-update (admm.cpp:66-101) on odd/even mixed grids
    for i, (shape, n) in enumerate([((4, 6, 5), 1), ((5, 4, 6), 2), ((8, 8, 8), 3)]):
        v, b = random_field(shape, 110 + i, 1.0), random_field(shape, 120 + i, 1.0)
        out[f"wu{i}_v"], out[f"wu{i}_b"] = v, b
        out[f"wu{i}_out"] = ref.w_update(v, b, abi.solver_cfg(order=n, lambda_=2.0, theta=0.1))
        out[f"wu{i}_energy"] = np.array(ref.regulariser_energy(v, n))
    # field ops (volume.cpp)
    img = random_volume((7, 9, 8), 130)
    disp = random_field((7, 9, 8), 131, 1.5)
    out.update(f_img=img, f_disp=disp)
    out["f_warp"] = ref.warp_image(img, disp)
    out["f_grad"] = ref.image_gradient(img)
    a = smooth_random_field((7, 9, 8), 132, 0.4, ref)
    out["f_phi"] = a
    out["f_compose"] = ref.compose_deformation(a, disp * np.float32(0.3))
    out["f_det"] = ref.jacobian_determinant(disp * np.float32(0.5))
    st = ref.jacobian_stats(disp * np.float32(0.5))
    out["f_det_stats"] = np.array([st.nonpositive, st.interior, st.min_det, st.pct_nonpositive])
    oa, ob = ref.normalize_intensity_pair(img * 3 - 1, random_volume((7, 9, 8), 133, 2.0, 5.0))
    out["f_norm_a"], out["f_norm_b"] = oa, ob
    out["f_smooth"] = ref.binomial_smooth(img)
    out["f_down"] = ref.downsample(img)
    out["f_up"] = ref.upsample_velocity(random_field((4, 5, 4), 134, 1.0), (7, 9, 8))
    out["f_up_in"] = random_field((4, 5, 4), 134, 1.0)
    # solve_velocity (admm.cpp:252-314), 10^3, 12 iterations, objective logged
    f, m = synth.make_pair(1, 140, (10, 10, 10))
    out.update(sv_target=f, sv_warped=m)
    for dt in (1, 2):
        cfg = abi.solver_cfg(data_term=dt, order=2, lambda_=0.3, theta=0.2, max_iters=12, log_objective=True)
        v, d = ref.solve_velocity(f, m, cfg)
        out[f"sv_v_s{dt}"] = v
        out[f"sv_obj_s{dt}"] = d["objective"]
        out[f"sv_res_s{dt}"] = d["constraint_residual"]
        out[f"sv_change_s{dt}"] = np.array(d["final_change"])
    # register_pair (registration.cpp:180-283): levels 1 and a 2-level capped run
    f, m = synth.make_pair(1, 150, (16, 16, 16))
    out.update(rp_target=f, rp_source=m)
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=20, log_objective=False)
    phi, warped, res = ref.register_pair(f, m, abi.reg_cfg(s, 1, (3,), (20,)))
    out["rp1_phi"], out["rp1_warped"] = phi, warped
    lg = abi.level_logs(res)[0]
    out["rp1_log"] = np.array([res.velocity_count] + lg["mean_sad"] + lg["solver_iterations"], np.float64)
    cfg2 = ref.make_registration_config(abi.DREG_PROFILE_CAPPED, abi.solver_cfg(data_term=1, order=2, lambda_=5.0,
                                                                               theta=0.05, log_objective=False), 2)
    phi, warped, res = ref.register_pair(f, m, cfg2)
    out["rp2_phi"], out["rp2_warped"] = phi, warped
    out["rp2_velocity_count"] = np.array(res.velocity_count)
    path = os.path.join(HERE, "ref_fixtures.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
