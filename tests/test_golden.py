"""Golden fixtures produced by the unmodified reference (tests/golden/make_golden.py).

backend "oracle": the plain-C restatement must reproduce every fixture BIT-EXACTLY
                  (same fp64 arithmetic, same FFT), which pins the oracle itself.
backend "gpu":    the sm_100a path within the tolerances of tests/test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

from conftest import max_abs, rel_l2
from paper_2109_12688_b200 import abi

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_fixtures.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(FIX))


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def lib(request, oracle):
    if request.param == "oracle":
        return oracle
    return request.getfixturevalue("ctx")


def is_oracle(lib):
    return lib.__class__.__name__ == "CpuLib"


def close(lib, out, ref, rtol_gpu=4e-7):
    if is_oracle(lib):
        assert np.array_equal(np.asarray(out), np.asarray(ref)), max_abs(out, ref)
    else:
        ref = np.asarray(ref, np.float64)
        tol = rtol_gpu * np.maximum(np.abs(ref), 1.0)
        assert np.all(np.abs(np.asarray(out, np.float64) - ref) <= tol), max_abs(out, ref)


def test_symbol(gold):
    from paper_2109_12688_b200 import dreg

    for n, dims in [(1, (4, 6, 5)), (2, (8, 4, 6)), (3, (5, 5, 4))]:
        # the C ABI's host helper; fp64 like the reference (regularizer.cpp:51-79)
        try:
            out = dreg.laplacian_symbol(n, dims)
        except ImportError:
            pytest.skip("libdreg_cuda.so not built")
        assert np.allclose(out, gold[f"symbol_n{n}"], rtol=1e-15, atol=1e-15)


def test_oracle_symbol(oracle, gold):
    for n, dims in [(1, (4, 6, 5)), (2, (8, 4, 6)), (3, (5, 5, 4))]:
        assert np.array_equal(oracle.laplacian_symbol(n, dims), gold[f"symbol_n{n}"])


@pytest.mark.parametrize("dt", [1, 2])
def test_v_update(lib, gold, dt):
    g = gold
    out = lib.v_update(g["vu_target"], g["vu_warped"], g["vu_grad"], g["vu_w_hat"], g["vu_b_hat"],
                       abi.solver_cfg(data_term=dt, theta=0.07))
    close(lib, out, g[f"vu_out_s{dt}"], rtol_gpu=1e-6)


@pytest.mark.parametrize("i,n", [(0, 1), (1, 2), (2, 3)])
def test_w_update_and_energy(lib, gold, i, n):
    out = lib.w_update(gold[f"wu{i}_v"], gold[f"wu{i}_b"], abi.solver_cfg(order=n, lambda_=2.0, theta=0.1))
    ref = gold[f"wu{i}_out"]
    e = lib.regulariser_energy(gold[f"wu{i}_v"], n)
    if is_oracle(lib):
        assert np.array_equal(out, ref)
        assert e == float(gold[f"wu{i}_energy"])
    else:
        assert max_abs(out, ref) <= 1e-5 * np.abs(ref).max()
        assert abs(e - float(gold[f"wu{i}_energy"])) <= 2e-6 * abs(float(gold[f"wu{i}_energy"]))


def test_field_ops(lib, gold):
    g = gold
    close(lib, lib.warp_image(g["f_img"], g["f_disp"]), g["f_warp"])
    close(lib, lib.image_gradient(g["f_img"]), g["f_grad"])
    close(lib, lib.compose_deformation(g["f_phi"], g["f_disp"] * np.float32(0.3)), g["f_compose"])
    close(lib, lib.jacobian_determinant(g["f_disp"] * np.float32(0.5)), g["f_det"], rtol_gpu=2e-6)
    st = lib.jacobian_stats(g["f_disp"] * np.float32(0.5))
    ref = g["f_det_stats"]
    assert st.nonpositive == int(ref[0]) and st.interior == int(ref[1])
    assert abs(st.min_det - ref[2]) <= (0 if is_oracle(lib) else 1e-6)
    a, b = lib.normalize_intensity_pair(g["f_img"] * 3 - 1, _vol133())
    close(lib, a, g["f_norm_a"])
    close(lib, b, g["f_norm_b"])
    close(lib, lib.binomial_smooth(g["f_img"]), g["f_smooth"])
    close(lib, lib.downsample(g["f_img"]), g["f_down"])
    close(lib, lib.upsample_velocity(g["f_up_in"], (7, 9, 8)), g["f_up"])  # Dims3 (x, y, z)


def _vol133():
    from conftest import random_volume

    return random_volume((7, 9, 8), 133, 2.0, 5.0)


@pytest.mark.parametrize("dt", [1, 2])
def test_solve_velocity(lib, gold, dt):
    cfg = abi.solver_cfg(data_term=dt, order=2, lambda_=0.3, theta=0.2, max_iters=12, log_objective=True)
    v, d = lib.solve_velocity(gold["sv_target"], gold["sv_warped"], cfg)
    if is_oracle(lib):
        assert np.array_equal(v, gold[f"sv_v_s{dt}"])
        assert np.array_equal(d["objective"], gold[f"sv_obj_s{dt}"])
        assert np.array_equal(d["constraint_residual"], gold[f"sv_res_s{dt}"])
        assert d["final_change"] == float(gold[f"sv_change_s{dt}"])
    else:
        assert max_abs(v, gold[f"sv_v_s{dt}"]) <= 1e-4
        assert np.allclose(d["objective"], gold[f"sv_obj_s{dt}"], rtol=1e-4)
        assert np.allclose(d["constraint_residual"], gold[f"sv_res_s{dt}"], rtol=1e-4, atol=1e-7)


def test_register_pair_levels1(lib, gold):
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=20, log_objective=False)
    phi, warped, res = lib.register_pair(gold["rp_target"], gold["rp_source"], abi.reg_cfg(s, 1, (3,), (20,)))
    lg = abi.level_logs(res)[0]
    log = np.array([res.velocity_count] + lg["mean_sad"] + lg["solver_iterations"], np.float64)
    if is_oracle(lib):
        assert np.array_equal(phi, gold["rp1_phi"]) and np.array_equal(warped, gold["rp1_warped"])
        assert np.array_equal(log, gold["rp1_log"])
    else:
        assert res.velocity_count == int(gold["rp1_log"][0])
        assert max_abs(phi, gold["rp1_phi"]) <= 1e-3 and rel_l2(phi, gold["rp1_phi"]) <= 1e-4
        assert np.allclose(log, gold["rp1_log"], rtol=1e-4)


def test_register_pair_two_levels(lib, gold):
    cfg = lib.make_registration_config(
        abi.DREG_PROFILE_CAPPED,
        abi.solver_cfg(data_term=1, order=2, lambda_=5.0, theta=0.05, log_objective=False), 2)
    phi, warped, res = lib.register_pair(gold["rp_target"], gold["rp_source"], cfg)
    assert res.velocity_count == int(gold["rp2_velocity_count"])
    if is_oracle(lib):
        assert np.array_equal(phi, gold["rp2_phi"]) and np.array_equal(warped, gold["rp2_warped"])
    else:
        assert max_abs(phi, gold["rp2_phi"]) <= 1e-3 and rel_l2(phi, gold["rp2_phi"]) <= 1e-4
