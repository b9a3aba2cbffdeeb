"""GPU parity: the sm_100a path (C ABI via paper_2109_12688_b200.dreg) against the CPU
oracle (oracle/dreg_oracle.c, itself pinned bit-exact to the unmodified reference in
tests/test_oracle_pin.py) on identical seeded inputs.

Tolerances (BASELINE.json north_star): displacement fields max-abs <= 1e-3 voxel and
relative L2 <= 1e-4; folding counts (det J <= 0) exactly equal.  Point-wise fp64
building blocks are held to fp32 rounding (a few ulp); the fp32 spectral solve to
1e-5 * max|ref| like the reference's own w-update pin (test_admm.cpp:184-211).
"""
import json
import os

import numpy as np
import pytest

from conftest import max_abs, random_field, random_volume, rel_l2, smooth_random_field
from paper_2109_12688_b200 import abi, dreg, synth

pytestmark = pytest.mark.gpu

PHI_MAX_ABS = 1e-3
PHI_REL_L2 = 1e-4


def ulp_close(a, b, rel=4e-7, abs_=1e-30):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    tol = rel * np.maximum(np.abs(b), 1.0) + abs_
    return bool(np.all(np.abs(a - b) <= tol))


# ---- building blocks (volume.cpp / admm.cpp point-wise) ---------------------------
@pytest.mark.parametrize("shape", [(8, 8, 8), (5, 7, 6), (16, 32, 24)])
def test_warp_image(ctx, oracle, shape):
    img = random_volume(shape, 21)
    disp = random_field(shape, 22, 1.5)  # test_volume.cpp:79-97 (amplitude 1.5)
    assert ulp_close(ctx.warp_image(img, disp), oracle.warp_image(img, disp))


def test_identity_warp_bit_exact(ctx):
    img = random_volume((8, 8, 8), 21)
    out = ctx.warp_image(img, np.zeros(img.shape + (3,), np.float32))
    assert np.array_equal(out, img)  # test_volume.cpp:72-77


@pytest.mark.parametrize("shape", [(8, 8, 8), (2, 3, 5), (16, 32, 24)])
def test_image_gradient(ctx, oracle, shape):
    img = random_volume(shape, 31)
    assert ulp_close(ctx.image_gradient(img), oracle.image_gradient(img))


def test_compose(ctx, oracle):
    shape = (8, 8, 8)
    a = smooth_random_field(shape, 51, 0.4, oracle)
    b = smooth_random_field(shape, 52, 0.4, oracle)
    assert ulp_close(ctx.compose_deformation(a, b), oracle.compose_deformation(a, b))
    zero = np.zeros_like(b)
    assert np.array_equal(ctx.compose_deformation(a, zero), a)  # test_volume.cpp:148-160


@pytest.mark.parametrize("shape", [(8, 8, 8), (16, 32, 24)])
def test_jacobian(ctx, oracle, shape):
    u = random_field(shape, 61, 0.6)
    det = ctx.jacobian_determinant(u)
    assert ulp_close(det, oracle.jacobian_determinant(u), rel=2e-6)
    st, so = ctx.jacobian_stats(u), oracle.jacobian_stats(u)
    assert st.nonpositive == so.nonpositive and st.interior == so.interior
    assert abs(st.min_det - so.min_det) <= 1e-6 * max(1.0, abs(so.min_det))


@pytest.mark.parametrize("data_term", [1, 2])
@pytest.mark.parametrize("theta", [0.03, 0.12])
def test_v_update(ctx, oracle, data_term, theta):
    shape = (10, 10, 10)  # acceptance crit 2 (acceptance_main.cpp:120-159)
    s0 = int(theta * 1000)
    t, w = random_volume(shape, s0), random_volume(shape, s0 + 1)
    g, wh, bh = random_field(shape, s0 + 2, 1.0), random_field(shape, s0 + 3, 1.0), random_field(shape, s0 + 4, 1.0)
    cfg = abi.solver_cfg(data_term=data_term, theta=theta)
    assert ulp_close(ctx.v_update(t, w, g, wh, bh, cfg), oracle.v_update(t, w, g, wh, bh, cfg), rel=1e-6)


def test_normalize_smooth_sad(ctx, oracle):
    a = random_volume((12, 20, 16), 71, -3.0, 7.0)
    b = random_volume((12, 20, 16), 72, -1.0, 9.0)
    oa, ob = ctx.normalize_intensity_pair(a, b)
    ra, rb = oracle.normalize_intensity_pair(a, b)
    assert np.array_equal(oa, ra) and np.array_equal(ob, rb)
    assert ulp_close(ctx.binomial_smooth(a), oracle.binomial_smooth(a))
    assert abs(ctx.mean_sad(a, b) - oracle.mean_sad(a, b)) <= 1e-12 * oracle.mean_sad(a, b)


def test_downsample_upsample(ctx, oracle):
    a = random_volume((9, 12, 7), 81)
    assert ulp_close(ctx.downsample(a), oracle.downsample(a))
    v = random_field((5, 6, 4), 82, 1.0)
    assert ulp_close(ctx.upsample_velocity(v, (9, 11, 10)), oracle.upsample_velocity(v, (9, 11, 10)))


# ---- spectral w-update (admm.cpp:66-101) -------------------------------------------
W_SHAPES = [(4, 4, 4), (4, 6, 4), (4, 4, 5), (6, 5, 7), (8, 8, 8), (12, 10, 9), (16, 16, 16),
            (32, 64, 64), (64, 128, 128), (30, 36, 42), (16, 20, 96),
            # every (Nz, Ny) of the register-blocked plane kernel (plane_fast.cuh)
            (64, 64, 16), (128, 64, 8), (128, 128, 8)]


@pytest.mark.parametrize("shape", W_SHAPES)
@pytest.mark.parametrize("order", [1, 2, 3])
def test_w_update(ctx, oracle, shape, order):
    v = random_field(shape, 40 + order, 1.0)
    bh = random_field(shape, 50 + order, 1.0)
    cfg = abi.solver_cfg(order=order, lambda_=2.0, theta=0.1)
    out, ref = ctx.w_update(v, bh, cfg), oracle.w_update(v, bh, cfg)
    assert max_abs(out, ref) <= 1e-5 * np.abs(ref).max(), max_abs(out, ref)


@pytest.mark.parametrize("order", [4, 5, 6])
def test_w_update_high_order(ctx, oracle, order):
    """Orders above 3 take the run-time-order multiplier of the plane kernels."""
    shape = (64, 128, 16)
    v, bh = random_field(shape, 70 + order, 1.0), random_field(shape, 80 + order, 1.0)
    cfg = abi.solver_cfg(order=order, lambda_=0.5, theta=0.1)
    out, ref = ctx.w_update(v, bh, cfg), oracle.w_update(v, bh, cfg)
    assert max_abs(out, ref) <= 1e-5 * np.abs(ref).max(), max_abs(out, ref)


def test_w_update_lambda0_passthrough(ctx):
    v, bh = random_field((6, 6, 6), 60, 1.0), random_field((6, 6, 6), 61, 1.0)
    out = ctx.w_update(v, bh, abi.solver_cfg(order=2, lambda_=0.0, theta=0.1))
    assert max_abs(out, v.astype(np.float64) + bh) <= 1e-5  # test_admm.cpp:213-227


@pytest.mark.parametrize("shape", [(4, 4, 4), (6, 5, 7), (32, 64, 64), (64, 128, 16), (128, 128, 8)])
@pytest.mark.parametrize("order", [1, 2, 3])
def test_regulariser_energy(ctx, oracle, shape, order):
    w = random_field(shape, 90 + order, 1.0)
    e, r = ctx.regulariser_energy(w, order), oracle.regulariser_energy(w, order)
    assert abs(e - r) <= 2e-6 * abs(r)


def test_trilinear_sample_points(ctx, reference):
    """volume.hpp:107,110 (trilinear_sample) on the device vs the reference's own
    function: fp64 lerps, so equal to ~1e-15 relative (device FMA contraction)."""
    from test_oracle_pin import _points

    shape = (7, 9, 8)
    img, fld = random_volume(shape, 61), random_field(shape, 62, 2.0)
    pts = _points(shape, 63)
    for f in (img, fld):
        a, b = ctx.trilinear_sample(f, pts), reference.trilinear_sample(f, pts)
        assert np.allclose(a, b, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("s", [1, 2])
def test_data_term_value(ctx, reference, s):
    """admm.cpp:239-250 on the device (fp64 reduction) vs the reference."""
    shape = (16, 24, 20)
    t, w = random_volume(shape, 64), random_volume(shape, 65)
    g, v = random_field(shape, 66, 1.0), random_field(shape, 67, 0.5)
    a, b = ctx.data_term_value(t, w, g, v, s), reference.data_term_value(t, w, g, v, s)
    assert abs(a - b) <= 1e-12 * abs(b)
    assert ctx.data_term_value(t, w, g, v, s) == a  # fixed-order reduction: run-to-run identical


# ---- solve_velocity (admm.cpp:252-314) ----------------------------------------------
@pytest.mark.parametrize("data_term", [1, 2])
@pytest.mark.parametrize("shape", [(16, 16, 16), (32, 64, 64)])
def test_solve_velocity(ctx, oracle, data_term, shape):
    f, m = synth.make_pair(1, 5, shape)
    cfg = abi.solver_cfg(data_term=data_term, order=2, lambda_=0.1, theta=1.0, max_iters=50, log_objective=True)
    v, d = ctx.solve_velocity(f, m, cfg)
    vo, do = oracle.solve_velocity(f, m, cfg)
    assert d["iterations"] == do["iterations"] == 50
    assert max_abs(v, vo) <= PHI_MAX_ABS and rel_l2(v, vo) <= PHI_REL_L2, (max_abs(v, vo), rel_l2(v, vo))
    assert np.allclose(d["constraint_residual"], do["constraint_residual"], rtol=1e-4, atol=1e-6)
    assert np.allclose(d["objective"], do["objective"], rtol=1e-4, atol=1e-8)
    assert abs(d["final_change"] - do["final_change"]) <= 1e-4 * max(do["final_change"], 1e-12)


@pytest.mark.parametrize("precision", [1, 2])
@pytest.mark.parametrize("shape", [(16, 16, 16), (16, 32, 64), (16, 24, 48)])
@pytest.mark.parametrize("data_term", [1, 2])
def test_velocity_independent_of_log_objective(ctx, precision, shape, data_term):
    """The logged objective's r2c(v_k) goes to a scratch spectrum, so v is bit-identical
    with log_objective on and off (the reference's solve does not depend on it,
    admm.cpp:288-292), for fp32 and fp64 spectral arithmetic and for the generic
    (M = 16, 48) and specialised (M = 64) x-pass."""
    f, m = synth.make_pair(1, 9, shape)
    ctx.set_precision(precision)
    try:
        on = abi.solver_cfg(data_term=data_term, order=2, lambda_=0.1, theta=1.0, max_iters=12, log_objective=True)
        off = abi.solver_cfg(data_term=data_term, order=2, lambda_=0.1, theta=1.0, max_iters=12, log_objective=False)
        v1, d1 = ctx.solve_velocity(f, m, on)
        v0, d0 = ctx.solve_velocity(f, m, off)
    finally:
        ctx.set_precision(0)
    assert np.array_equal(v0, v1)
    assert d1["objective"].shape == (12,) and np.all(np.isfinite(d1["objective"]))


@pytest.mark.parametrize("shape", [(16, 24, 48), (12, 20, 30)])
def test_long_solve_generic_width_precise(ctx, oracle, shape):
    """> 100 iterations at x extents the specialised x-pass does not cover (M = 48, 30):
    the auto policy runs the generic x-pass with fp64 butterflies (precise mode), and
    the 150-iteration accelerated solve stays within the 1e-4 contract of the oracle."""
    f, m = synth.make_pair(1, 13, shape)
    cfg = abi.solver_cfg(data_term=2, order=3, lambda_=0.05, theta=0.5, max_iters=150, log_objective=False)
    v, d = ctx.solve_velocity(f, m, cfg)
    vo, do = oracle.solve_velocity(f, m, cfg)
    print(f"{shape}: max-abs {max_abs(v, vo):.2e} rel-L2 {rel_l2(v, vo):.2e}")
    assert d["iterations"] == do["iterations"] == 150
    assert max_abs(v, vo) <= PHI_MAX_ABS and rel_l2(v, vo) <= PHI_REL_L2, (max_abs(v, vo), rel_l2(v, vo))


def test_solve_velocity_tol_early_exit(ctx, oracle):
    f, m = synth.make_pair(1, 6, (16, 16, 16))
    cfg = abi.solver_cfg(data_term=2, order=1, lambda_=2.0, theta=0.05, max_iters=200, tol=1e-4, log_objective=False)
    v, d = ctx.solve_velocity(f, m, cfg)
    vo, do = oracle.solve_velocity(f, m, cfg)
    assert d["converged"] and do["converged"]
    assert abs(d["iterations"] - do["iterations"]) <= 1
    assert max_abs(v, vo) <= PHI_MAX_ABS


def test_solve_identical_images_is_zero(ctx):
    img = random_volume((12, 12, 12), 3)
    cfg = abi.solver_cfg(data_term=1, order=1, lambda_=1.0, theta=0.1, max_iters=50, tol=1e-7)
    v, d = ctx.solve_velocity(img, img, cfg)
    assert np.abs(v).mean() <= 1e-4  # test_admm.cpp:250-266


# ---- register_pair (registration.cpp:180-283), levels = 1 ----------------------------
def _reg_parity(ctx, oracle, f, m, cfg):
    phi, warped, res = ctx.register_pair(f, m, cfg)
    phi_o, warped_o, res_o = oracle.register_pair(f, m, cfg)
    assert res.status == 0
    assert res.velocity_count == res_o.velocity_count
    lg, lo = abi.level_logs(res)[0], abi.level_logs(res_o)[0]
    assert lg["solver_iterations"] == lo["solver_iterations"]
    print(f"phi max-abs {max_abs(phi, phi_o):.3e} rel-L2 {rel_l2(phi, phi_o):.3e} velocity_count {res.velocity_count}")
    assert max_abs(phi, phi_o) <= PHI_MAX_ABS, max_abs(phi, phi_o)
    assert rel_l2(phi, phi_o) <= PHI_REL_L2, rel_l2(phi, phi_o)
    # per-warp mean SAD log (registration.cpp:247,262): fp32 spectral solve -> 1e-4 relative
    assert np.allclose(lg["mean_sad"], lo["mean_sad"], rtol=1e-4, atol=1e-9)
    assert ctx.jacobian_stats(phi).nonpositive == oracle.jacobian_stats(phi_o).nonpositive
    assert max_abs(warped, warped_o) <= 1e-3
    return phi, res


@pytest.mark.parametrize("data_term", [1, 2])
def test_register_small(ctx, oracle, data_term):
    f, m = synth.make_pair(1, 7, (16, 32, 32))
    s = abi.solver_cfg(data_term=data_term, order=2, lambda_=0.1, theta=1.0, max_iters=50, log_objective=False)
    _reg_parity(ctx, oracle, f, m, abi.reg_cfg(s, 1, (5,), (50,)))


def test_register_config1(ctx, oracle):
    c = synth.CONFIGS["config1"]
    f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
    _reg_parity(ctx, oracle, f, m, synth.config_cfg("config1"))


@pytest.mark.slow
@pytest.mark.parametrize("order", [1, 2, 3])
def test_register_config2(ctx, oracle, order):
    c = synth.CONFIGS["config2"]
    f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
    _reg_parity(ctx, oracle, f, m, synth.config_cfg("config2", order=order))


def test_batch_matches_single_and_is_deterministic(ctx):
    F, M = synth.make_batch(1, 300, 3, (16, 32, 32))
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=30, log_objective=False)
    cfg = abi.reg_cfg(s, 1, (4,), (30,))
    phis, warps, res = ctx.register_batch(list(F), list(M), cfg)
    for i in range(3):
        p1, w1, r1 = ctx.register_pair(F[i], M[i], cfg)
        assert np.array_equal(p1, phis[i]) and np.array_equal(w1, warps[i])
        assert r1.velocity_count == res[i].velocity_count
    phis2, _, _ = ctx.register_batch(list(F), list(M), cfg)
    assert all(np.array_equal(a, b) for a, b in zip(phis, phis2))


def test_device_batch_auto_chunks_match_single(ctx):
    """Device-resident batches run in launch chunks of up to 256 pairs (pick_chunk):
    260 pairs = 256 + 4.  Pairs on both sides of the chunk boundary give the same phi
    and warped image as registering them alone (tol = 0: the result of a pair does not
    depend on the batch it runs in)."""
    import torch

    n, shape = 260, (16, 32, 32)
    F, M = synth.make_batch(1, 500, n, shape)
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=20, log_objective=False)
    cfg = abi.reg_cfg(s, 1, (3,), (20,))
    N = int(np.prod(shape))
    dev = torch.device("cuda", 0)
    tgt = torch.from_numpy(F.reshape(n, N)).to(dev)
    src = torch.from_numpy(M.reshape(n, N)).to(dev)
    phi = torch.empty((n, 3, N), dtype=torch.float32, device=dev)
    warped = torch.empty((n, N), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    res = ctx.register_batch_device(n, tgt.data_ptr(), src.data_ptr(), shape[::-1], cfg, phi.data_ptr(),
                                    warped.data_ptr())
    torch.cuda.synchronize()
    assert all(r.status == 0 for r in res)
    ph = phi.cpu().numpy()
    wp = warped.cpu().numpy()
    for i in (0, 255, 256, 259):
        p1, w1, r1 = ctx.register_pair(F[i], M[i], cfg)
        assert r1.velocity_count == res[i].velocity_count
        assert np.array_equal(p1, np.moveaxis(ph[i].reshape(3, *shape), 0, -1)), i
        assert np.array_equal(w1, wp[i].reshape(shape)), i


def test_register_nonfinite_input_raises(ctx):
    f, m = synth.make_pair(1, 8, (16, 16, 16))
    m[3, 4, 5] = np.nan
    s = abi.solver_cfg(data_term=2, max_iters=5)
    with pytest.raises(dreg.NumericError):
        ctx.register_pair(f, m, abi.reg_cfg(s, 1, (2,), (5,)))


def test_register_invalid_config_raises(ctx):
    f, m = synth.make_pair(1, 8, (16, 16, 16))
    with pytest.raises(ValueError):
        ctx.register_pair(f, m, abi.reg_cfg(abi.solver_cfg(data_term=3), 1, (2,), (5,)))
    with pytest.raises(ValueError):
        ctx.register_pair(f, m, abi.reg_cfg(abi.solver_cfg(theta=0.0), 1, (2,), (5,)))
    with pytest.raises(ValueError):
        ctx.register_pair(f, m, abi.reg_cfg(abi.solver_cfg(), 1, (2,), (5,), warp_improvement_threshold=1.5))
    with pytest.raises(ValueError):
        ctx.register_pair(f[:3], m[:3], abi.reg_cfg(abi.solver_cfg(), 1, (2,), (5,)))


def test_identity_pair(ctx):
    f, _ = synth.make_pair(1, 9, (32, 32, 32))
    s = abi.solver_cfg(data_term=1, order=2, lambda_=5.0, theta=0.05, max_iters=10, log_objective=False)
    phi, warped, res = ctx.register_pair(f, f, abi.reg_cfg(s, 1, (5,), (10,)))
    assert np.abs(phi).mean() <= 0.05  # test_registration.cpp:197-210


# ---- pyramid: levels > 1 (registration.cpp:208-247, make_registration_config :62-83) ----
@pytest.mark.parametrize("levels,data_term", [(2, 2), (3, 1), (3, 2)])
def test_register_pyramid_capped(ctx, oracle, levels, data_term):
    f, m = synth.make_pair(1, 21, (32, 64, 64))
    s = abi.solver_cfg(data_term=data_term, order=2, lambda_=0.1 if data_term == 2 else 5.0,
                       theta=1.0 if data_term == 2 else 0.05, log_objective=False)
    cfg = oracle.make_registration_config(abi.DREG_PROFILE_CAPPED, s, levels)
    phi, warped, res = ctx.register_pair(f, m, cfg)
    phi_o, warped_o, res_o = oracle.register_pair(f, m, cfg)
    lg, lo = abi.level_logs(res), abi.level_logs(res_o)
    assert [l["dims"] for l in lg] == [l["dims"] for l in lo]
    assert [l["solver_iterations"] for l in lg] == [l["solver_iterations"] for l in lo]
    assert res.velocity_count == res_o.velocity_count
    print(f"levels {levels}: phi max-abs {max_abs(phi, phi_o):.3e} rel-L2 {rel_l2(phi, phi_o):.3e}")
    assert max_abs(phi, phi_o) <= PHI_MAX_ABS and rel_l2(phi, phi_o) <= PHI_REL_L2
    assert ctx.jacobian_stats(phi).nonpositive == oracle.jacobian_stats(phi_o).nonpositive
    for a, b in zip(lg, lo):
        assert np.allclose(a["mean_sad"], b["mean_sad"], rtol=1e-4, atol=1e-9)


def test_register_pyramid_converged_odd_dims(ctx, oracle):
    """converged profile (tol 0.01 early exit per solve) on odd extents (edge-replicated downsample)."""
    f, m = synth.make_pair(1, 22, (19, 21, 23))
    s = abi.solver_cfg(data_term=2, order=1, lambda_=0.5, theta=0.5, log_objective=False)
    cfg = oracle.make_registration_config(abi.DREG_PROFILE_CONVERGED, s, 2)
    cfg.max_warps_per_level[0] = 4
    cfg.max_warps_per_level[1] = 3
    phi, warped, res = ctx.register_pair(f, m, cfg)
    phi_o, warped_o, res_o = oracle.register_pair(f, m, cfg)
    lg, lo = abi.level_logs(res), abi.level_logs(res_o)
    assert res.velocity_count == res_o.velocity_count
    for a, b in zip(lg, lo):
        assert a["dims"] == b["dims"]
        assert all(abs(x - y) <= 1 for x, y in zip(a["solver_iterations"], b["solver_iterations"]))
    assert max_abs(phi, phi_o) <= PHI_MAX_ABS


def test_pyramid_batch_matches_single(ctx):
    F, M = synth.make_batch(1, 400, 3, (16, 32, 32))
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, log_objective=False)
    cfg = dreg.make_registration_config(abi.DREG_PROFILE_CAPPED, s, 2)
    phis, warps, res = ctx.register_batch(list(F), list(M), cfg)
    for i in range(3):
        p1, w1, r1 = ctx.register_pair(F[i], M[i], cfg)
        assert np.array_equal(p1, phis[i]) and r1.velocity_count == res[i].velocity_count


# ---- large planes (split three-pass yz kernel, radix-3 z axis) -------------------------
@pytest.mark.parametrize("shape", [(48, 64, 256), (96, 160, 64), (24, 320, 32)])
def test_w_update_split_plane(ctx, oracle, shape):
    """planes whose y*z complex exceeds one CTA's shared memory take the 3-pass path."""
    v, bh = random_field(shape, 77, 1.0), random_field(shape, 78, 1.0)
    cfg = abi.solver_cfg(order=2, lambda_=2.0, theta=0.1)
    out, ref = ctx.w_update(v, bh, cfg), oracle.w_update(v, bh, cfg)
    assert max_abs(out, ref) <= 1e-5 * np.abs(ref).max()
    e, r = ctx.regulariser_energy(v, 2), oracle.regulariser_energy(v, 2)
    assert abs(e - r) <= 2e-6 * abs(r)


@pytest.mark.slow
def test_w_update_config5_grid(ctx, oracle):
    """config 5 grid (Dims3{256,256,192}): 256 x 192 planes, radix-3 z axis, M = 256 x-pass."""
    shape = (192, 256, 256)
    v, bh = random_field(shape, 79, 1.0), random_field(shape, 80, 1.0)
    cfg = abi.solver_cfg(order=2, lambda_=0.1, theta=1.0)
    out, ref = ctx.w_update(v, bh, cfg), oracle.w_update(v, bh, cfg)
    assert max_abs(out, ref) <= 1e-5 * np.abs(ref).max()


@pytest.mark.slow
def test_register_config4_like(ctx, oracle):
    """config 4 settings (swirl phantom, n=3, lambda 0.05, theta 0.5, 15 fields x 200 iterations)
    on a 64^3 grid so the single-threaded oracle finishes; zero folding on both sides."""
    f, m = synth.make_pair(4, 4, (64, 64, 64))
    c = synth.CONFIGS["config4"]
    s = abi.solver_cfg(data_term=2, order=c["order"], lambda_=c["lambda_"], theta=c["theta"],
                       max_iters=c["iters"], log_objective=False)
    cfg = abi.reg_cfg(s, 1, (c["warps"],), (c["iters"],))
    phi, res = _reg_parity(ctx, oracle, f, m, cfg)
    assert ctx.jacobian_stats(phi).nonpositive == 0


@pytest.mark.slow
def test_register_config5_grid_short(ctx, oracle):
    """config 5 grid and phantom (Dims3{256,256,192}), 2 fields x 10 iterations."""
    c = synth.CONFIGS["config5"]
    f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=10, log_objective=False)
    _reg_parity(ctx, oracle, f, m, abi.reg_cfg(s, 1, (2,), (10,)))


@pytest.mark.slow
def test_config3_all_pairs_against_oracle_records(ctx):
    """Config 3: all 256 phantom pairs (seeds 1000..1255) registered in batches on the
    GPU vs the CPU oracle's recorded results (tests/golden/config3_oracle.json, made
    by tools/run_config3_oracle.py): identical velocity_count, solve count, per-solve
    iterations and folding counts; SAD logs within 1e-4; | |phi_gpu| - |phi_cpu| |
    <= 1e-4 |phi_cpu| (a necessary condition of the rel-L2 contract)."""
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "config3_oracle.json")
    rec = json.load(open(path))["pairs"]
    if len(rec) < 256:
        pytest.skip(f"oracle records incomplete ({len(rec)}/256)")
    cfg = synth.config_cfg("config3")
    shape = (64, 128, 128)
    mismatch = []
    for s0 in range(1000, 1256, 32):
        F, M = synth.make_batch(3, s0, 32, shape)
        phis, _, res = ctx.register_batch(list(F), list(M), cfg, want_warped=False)
        for i in range(32):
            r, o = res[i], rec[str(s0 + i)]
            lg = abi.level_logs(r)[0]
            js = ctx.jacobian_stats(phis[i])
            ok = (r.velocity_count == o["velocity_count"] and r.solves == o["solves"]
                  and lg["solver_iterations"] == o["solver_iterations"] and js.nonpositive == o["folding"]
                  and np.allclose(lg["mean_sad"], o["mean_sad"], rtol=1e-4))
            n_g = float(np.sqrt((phis[i].astype(np.float64) ** 2).sum()))
            n_c = float(np.sqrt(o["phi_sumsq"]))
            ok = ok and abs(n_g - n_c) <= 1e-4 * n_c
            if not ok:
                mismatch.append(s0 + i)
    assert not mismatch, mismatch


def _load_phi_fixture(name):
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "run_config3_phi", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "run_config3_phi.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.load(os.path.join(os.path.dirname(__file__), "golden", name))


@pytest.mark.slow
def test_config3_bench_path_full_fields(ctx):
    """The bench's own call -- all 256 config-3 pairs in ONE device-resident launch chunk
    (dreg_cuda_register_batch_device) -- against the oracle: every voxel of phi for the 8
    pairs in tests/golden/config3_phi (tools/run_config3_phi.py; quantised 2^-16) within
    max-abs 1e-3 and rel-L2 1e-4, and velocity / solve / iteration / folding counts of all
    256 pairs equal to tests/golden/config3_oracle.json."""
    import json

    torch = pytest.importorskip("torch")
    gold = os.path.join(os.path.dirname(__file__), "golden")
    rec = json.load(open(os.path.join(gold, "config3_oracle.json")))["pairs"]
    shape = (64, 128, 128)
    N = int(np.prod(shape))
    F, M = synth.make_batch(3, 1000, 256, shape)
    tgt = torch.from_numpy(F.reshape(256, N)).cuda()
    src = torch.from_numpy(M.reshape(256, N)).cuda()
    phi = torch.empty((256, 3, N), dtype=torch.float32, device="cuda")
    ctx.set_batch_chunk(0)  # library policy: one 256-pair chunk for a device-resident batch
    res = ctx.register_batch_device(256, tgt.data_ptr(), src.data_ptr(), shape[::-1], synth.config_cfg("config3"),
                                    phi.data_ptr(), 0)
    bad = []
    for i in range(256):
        r, o = res[i], rec[str(1000 + i)]
        lg = abi.level_logs(r)[0]
        if not (r.velocity_count == o["velocity_count"] and r.solves == o["solves"]
                and lg["solver_iterations"] == o["solver_iterations"] and r.folding_voxels == o["folding"]):
            bad.append(1000 + i)
    assert not bad, bad
    worst = (0.0, 0.0)
    for fn in sorted(os.listdir(os.path.join(gold, "config3_phi"))):
        seed = int(fn.split(".")[0])
        ref = _load_phi_fixture(os.path.join("config3_phi", fn))  # (z, y, x, 3)
        got = phi[seed - 1000].cpu().numpy().reshape(3, *shape).transpose(1, 2, 3, 0)
        e, r = max_abs(got, ref), rel_l2(got, ref)
        worst = (max(worst[0], e), max(worst[1], r))
        assert e <= PHI_MAX_ABS and r <= PHI_REL_L2, (seed, e, r)
    print(f"config 3 full fields (8 pairs): worst max-abs {worst[0]:.2e}, rel-L2 {worst[1]:.2e}")


# ---- robustness: grids through the generic kernels, mixed-validity batches --------------
@pytest.mark.parametrize("shape", [(8, 12, 20), (10, 16, 48), (12, 20, 96), (16, 16, 160), (4, 4, 4)])
def test_register_generic_grids(ctx, oracle, shape):
    """non-power-of-two x extents (generic x-pass), odd y/z (generic plane), tiny grids."""
    f, m = synth.make_pair(1, 23, shape)
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.2, theta=0.5, max_iters=30, log_objective=False)
    _reg_parity(ctx, oracle, f, m, abi.reg_cfg(s, 1, (3,), (30,)))


def test_register_cap_edge_cases(ctx, reference):
    """registration.cpp:182-198,250: a negative warp cap runs no warps (and its level's
    ADMM cap is never validated), caps above the old 64 are accepted, and > 10 levels
    fail with the reference's 'dims too small' on any grid one device can hold."""
    f, m = synth.make_pair(1, 21, (16, 16, 16))
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=10, log_objective=False)
    for cfg in (abi.reg_cfg(s, 2, (-3, 2), (0, 10)), abi.reg_cfg(s, 1, (100,), (3,))):
        cfg.warp_improvement_threshold = 1e-9
        phi, _, res = ctx.register_pair(f, m, cfg)
        phi_r, _, res_r = reference.register_pair(f, m, cfg)
        assert res.velocity_count == res_r.velocity_count
        assert abi.level_logs(res)[0]["warps"] == abi.level_logs(res_r)[0]["warps"]
        assert max_abs(phi, phi_r) <= PHI_MAX_ABS and rel_l2(phi, phi_r) <= PHI_REL_L2
    bad = abi.reg_cfg(s, 1, (2,), (0,))  # a level that runs a solve with max_iters 0
    with pytest.raises(ValueError):
        ctx.register_pair(f, m, bad)
    with pytest.raises(Exception, match="max_iters"):
        reference.register_pair(f, m, bad)
    with pytest.raises(ValueError):
        ctx.register_pair(f, m, abi.reg_cfg(s, 1, (2,), (10,)), spacing=(1.0, 0.0, 1.0))


def test_batch_isolates_bad_pair(ctx, oracle):
    """a NaN pair fails alone (status DREG_NUMERIC) and leaves its batch mates intact."""
    F, M = synth.make_batch(1, 500, 3, (16, 32, 32))
    M[1, 2, 3, 4] = np.nan
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=20, log_objective=False)
    cfg = abi.reg_cfg(s, 1, (3,), (20,))
    with pytest.raises(dreg.NumericError) as ei:
        ctx.register_batch(list(F), list(M), cfg)
    phis_e, _, res_e = ei.value.results  # the other pairs' outputs survive the exception
    assert [r.status for r in res_e] == [0, abi.DREG_NUMERIC, 0]
    import ctypes as C

    n = 3
    res = (abi.PairResult * n)()
    phis = [np.zeros((16, 32, 32, 3), np.float32) for _ in range(n)]
    Fp = C.POINTER(C.c_float)
    T = (Fp * n)(*[np.ascontiguousarray(F[i]).ctypes.data_as(Fp) for i in range(n)])
    S = (Fp * n)(*[np.ascontiguousarray(M[i]).ctypes.data_as(Fp) for i in range(n)])
    P = (Fp * n)(*[p.ctypes.data_as(Fp) for p in phis])
    st = ctx.lib.dreg_cuda_register_batch(ctx.h, n, T, S, abi.Dims3(32, 32, 16), abi.Spacing3(1, 1, 1),
                                          C.byref(cfg), P, None, res)
    assert st == abi.DREG_NUMERIC
    assert [r.status for r in res] == [0, abi.DREG_NUMERIC, 0]
    for i in (0, 2):
        po, _, _ = oracle.register_pair(F[i], M[i], cfg)
        assert max_abs(phis[i], po) <= PHI_MAX_ABS
        assert np.array_equal(phis_e[i], phis[i])


@pytest.mark.slow
def test_register_config4_full_against_oracle_record(ctx):
    """Full config 4 (128^3 swirl, n = 3, 15 fields x 200 iterations; auto precise mode) vs
    the oracle's record (tests/golden/config4_oracle.json + a [::4]^3 phi subsample, made by
    tools/run_config4_oracle.py, 23 CPU-minutes): identical velocity / solve / folding
    counts, SAD log within 1e-4, phi within the contract on the subsample."""
    gold = os.path.join(os.path.dirname(__file__), "golden")
    rec = json.load(open(os.path.join(gold, "config4_oracle.json")))
    sub = np.load(os.path.join(gold, "config4_phi_sub4.npz"))["phi"]
    c = synth.CONFIGS["config4"]
    f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
    phi, warped, res = ctx.register_pair(f, m, synth.config_cfg("config4"))
    assert res.status == 0
    assert res.velocity_count == rec["velocity_count"] and res.solves == rec["solves"]
    assert np.allclose(abi.level_logs(res)[0]["mean_sad"], rec["mean_sad"], rtol=1e-4, atol=1e-9)
    js = ctx.jacobian_stats(phi)
    print(f"config4 folding {js.nonpositive} (oracle {rec['folding']}) min det {js.min_det:.4f} "
          f"(oracle {rec['min_det']:.4f}) sub max-abs {max_abs(phi[::4, ::4, ::4], sub):.2e} "
          f"rel-L2 {rel_l2(phi[::4, ::4, ::4], sub):.2e}")
    assert js.nonpositive == rec["folding"]
    assert abs(js.min_det - rec["min_det"]) <= 1e-3
    assert max_abs(phi[::4, ::4, ::4], sub) <= PHI_MAX_ABS
    assert rel_l2(phi[::4, ::4, ::4], sub) <= PHI_REL_L2


@pytest.mark.slow
def test_register_config5_full_against_oracle_record(ctx):
    """Full config 5 (256 x 256 x 192 texture, n = 2, 10 fields x 50 iterations; the
    split three-pass plane path) vs the oracle's record (tests/golden/config5_oracle.json
    + a [::8]^3 phi subsample, made by tools/run_config5_oracle.py): identical velocity /
    solve / folding counts, SAD log within 1e-4, phi within the contract on the
    subsample."""
    gold = os.path.join(os.path.dirname(__file__), "golden")
    if not os.path.exists(os.path.join(gold, "config5_oracle.json")):
        pytest.skip("config-5 oracle record not generated (tools/run_config5_oracle.py)")
    rec = json.load(open(os.path.join(gold, "config5_oracle.json")))
    sub = np.load(os.path.join(gold, "config5_phi_sub8.npz"))["phi"]
    c = synth.CONFIGS["config5"]
    f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
    phi, warped, res = ctx.register_pair(f, m, synth.config_cfg("config5"))
    assert res.status == 0
    assert res.velocity_count == rec["velocity_count"] and res.solves == rec["solves"]
    assert np.allclose(abi.level_logs(res)[0]["mean_sad"], rec["mean_sad"], rtol=1e-4, atol=1e-9)
    js = ctx.jacobian_stats(phi)
    print(f"config5 folding {js.nonpositive} (oracle {rec['folding']}) min det {js.min_det:.4f} "
          f"(oracle {rec['min_det']:.4f}) sub max-abs {max_abs(phi[::8, ::8, ::8], sub):.2e} "
          f"rel-L2 {rel_l2(phi[::8, ::8, ::8], sub):.2e}")
    assert js.nonpositive == rec["folding"]
    assert abs(js.min_det - rec["min_det"]) <= 1e-3
    assert max_abs(phi[::8, ::8, ::8], sub) <= PHI_MAX_ABS
    assert rel_l2(phi[::8, ::8, ::8], sub) <= PHI_REL_L2


@pytest.mark.parametrize("shape", [(64, 128, 128), (32, 64, 64)])
def test_pipelined_xpass_bit_identical_to_one_tile_kernel(shape):
    """The warp-specialised persistent x-pass (default for M in {64, 128}) and the
    one-tile-per-CTA kernel (DREG_PIPE=0) produce bit-identical phi."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r)\n"
            "from paper_2109_12688_b200 import dreg, synth\n"
            "F, M = synth.make_batch(3, 1000, 3, %r)\n"
            "cfg = synth.config_cfg('config3')\n"
            "with dreg.Context(0) as ctx:\n"
            "    phis, _, res = ctx.register_batch(list(F), list(M), cfg, want_warped=False)\n"
            "h = hashlib.sha256(b''.join(np.ascontiguousarray(p).tobytes() for p in phis))\n"
            "print(h.hexdigest(), [r.velocity_count for r in res])\n") % (root, shape)
    outs = []
    for pipe in ("0", "1"):
        env = dict(os.environ, DREG_PIPE=pipe, DREG_SS="0")  # the real-space-state iteration
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs


def test_cluster_plane_kernel_matches_split_path():
    """The 2-CTA cluster / DSMEM plane kernels (plane_cluster.cu: DREG_CLUSTER=1 register-blocked, the
    default on the config-5 plane; 2 generic) compute the same w-update as the 3-pass split
    (DREG_CLUSTER=0) on the config-5 plane (256 x 192) within fp32 rounding."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "from paper_2109_12688_b200 import abi, dreg\n"
            "rng = np.random.default_rng(7)\n"
            "v = rng.standard_normal((192, 256, 32, 3)).astype(np.float32)\n"
            "b = rng.standard_normal((192, 256, 32, 3)).astype(np.float32)\n"
            "cfg = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=50)\n"
            "with dreg.Context(0) as ctx:\n"
            "    w = ctx.w_update(v, b, cfg)\n"
            "np.save(sys.argv[1], w)\n") % root
    import tempfile

    outs = []
    with tempfile.TemporaryDirectory() as td:
        for flag in ("0", "1", "2"):  # 3-pass split, register-blocked cluster kernel, generic cluster kernel
            path = os.path.join(td, f"w{flag}.npy")
            r = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, DREG_CLUSTER=flag),
                               capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
    scale = float(np.abs(outs[0]).max())
    print(f"cluster vs split w-update: max-abs {max_abs(outs[1], outs[0]):.3e} / {max_abs(outs[2], outs[0]):.3e} "
          f"(max|w| {scale:.3f})")
    assert max_abs(outs[1], outs[0]) <= 1e-5 * scale
    assert max_abs(outs[2], outs[0]) <= 1e-5 * scale


def test_cluster_plane_kernel_precise_matches_split_path():
    """The fp64 instance of the cluster plane kernel (128 x 128 planes, precise mode: config 4) against
    the generic fp64 3-pass split: same reference multiplier expression, fp64 transforms in a different
    order -- the w-updates agree to ~1e-13 relative."""
    import subprocess
    import sys
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "from paper_2109_12688_b200 import abi, dreg\n"
            "rng = np.random.default_rng(11)\n"
            "v = rng.standard_normal((128, 128, 16, 3)).astype(np.float32)\n"
            "b = rng.standard_normal((128, 128, 16, 3)).astype(np.float32)\n"
            "cfg = abi.solver_cfg(data_term=2, order=3, lambda_=0.05, theta=0.5, max_iters=200)\n"
            "with dreg.Context(0) as ctx:\n"
            "    ctx.set_precision(2)\n"
            "    w = ctx.w_update(v, b, cfg)\n"
            "np.save(sys.argv[1], w)\n") % root
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for flag in ("0", "1"):
            path = os.path.join(td, f"w{flag}.npy")
            r = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, DREG_CLUSTER=flag),
                               capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
    scale = float(np.abs(outs[0]).max())
    print(f"precise cluster vs split w-update: max-abs {max_abs(outs[1], outs[0]):.3e} (max|w| {scale:.3f})")
    assert max_abs(outs[1], outs[0]) <= 2e-7 * scale  # both round the same fp64 result to fp32


def test_pipelined_xpass_m256_bit_identical_to_one_tile_kernel():
    """M = 256: the pipelined x-pass with its two-buffer ring (DREG_PIPE256=1, default) and the
    one-tile-per-CTA kernel give bit-identical phi."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r)\n"
            "from paper_2109_12688_b200 import abi, dreg, synth\n"
            "F, M = synth.make_batch(3, 1000, 2, (6, 48, 256))\n"
            "s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=12, tol=0.0, log_objective=False)\n"
            "cfg = abi.reg_cfg(s, 1, (2,), (12,))\n"
            "with dreg.Context(0) as ctx:\n"
            "    phis, _, res = ctx.register_batch(list(F), list(M), cfg, want_warped=False)\n"
            "h = hashlib.sha256(b''.join(np.ascontiguousarray(p).tobytes() for p in phis))\n"
            "print(h.hexdigest(), [r.velocity_count for r in res])\n") % root
    outs = []
    for flag in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, DREG_PIPE256=flag), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs


# ---- spectral-state iteration (plane_fast.cuh MODE 2 + X_SS / X_SSN) -------------------
_SS_CODE = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r)\n"
            "from paper_2109_12688_b200 import dreg, synth\n"
            "F, M = synth.make_batch(3, 1000, 3, %r)\n"
            "cfg = synth.config_cfg('config3')\n"
            "cfg.max_warps_per_level[0] = 3\n"
            "with dreg.Context(0) as ctx:\n"
            "    phis, _, res = ctx.register_batch(list(F), list(M), cfg, want_warped=False)\n"
            "h = hashlib.sha256(b''.join(np.ascontiguousarray(p).tobytes() for p in phis))\n"
            "print(h.hexdigest(), [r.velocity_count for r in res])\n")


def _digest_under(env_extra, shape=(64, 128, 128)):
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", _SS_CODE % (root, shape)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_spectral_state_variants_bit_identical():
    """The spectral-state x-pass gives the same bits with and without the change norm
    (X_SS reads / writes v every iteration, X_SSN only writes the last one), pipelined or
    one tile per CTA or another warp split: the variants only move data differently."""
    base = _digest_under({})
    assert _digest_under({"DREG_SS_CHG": "1"}) == base
    assert _digest_under({"DREG_PIPE_SS": "3"}) == base
    assert _digest_under({"DREG_PIPE_SS": "80841"}) == base


@pytest.mark.parametrize("shape", [(64, 128, 128), (64, 64, 64)])
def test_spectral_state_matches_real_space_state(shape):
    """Same accelerated-ADMM recurrence (admm.cpp:275-308) carried as Fourier-domain iterates:
    against the real-space-state kernels (DREG_SS=0) the registrations agree far inside the
    parity contract (both are fp32 evaluations of the reference's fp64 arithmetic)."""
    F, M = synth.make_batch(3, 1000, 2, shape)
    cfg = synth.config_cfg("config3")
    cfg.max_warps_per_level[0] = 3
    out = {}
    for ss in ("1", "0"):
        os.environ["DREG_SS"] = ss
        try:
            with dreg.Context(0) as c2:
                phis, _, res = c2.register_batch(list(F), list(M), cfg, want_warped=False)
        finally:
            os.environ.pop("DREG_SS", None)
        out[ss] = (phis, [r.velocity_count for r in res])
    assert out["1"][1] == out["0"][1]
    for a, b in zip(out["1"][0], out["0"][0]):
        print(f"spectral vs real-space state: phi max-abs {max_abs(a, b):.3e} rel-L2 {rel_l2(a, b):.3e}")
        assert max_abs(a, b) <= 2e-4 and rel_l2(a, b) <= 5e-5


@pytest.mark.parametrize("tol", [0.0, 5e-5])
def test_register_spectral_state_grid(ctx, oracle, tol):
    """64^3 (a grid the spectral-state kernels cover) against the oracle, without a tolerance
    (X_SSN: v only written by the last iteration) and with one (X_SS: change norm, per-pair
    early exit at the oracle's iteration counts)."""
    f, m = synth.make_pair(2, 5, (64, 64, 64))
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=50, tol=tol, log_objective=False)
    phi, res = _reg_parity(ctx, oracle, f, m, abi.reg_cfg(s, 1, (4,), (50,)))
    if tol > 0:  # the tolerance stops the last solve inside the spectral-state loop (oracle: [50, 50, 50, 2])
        assert any(1 < it < 50 for it in abi.level_logs(res)[0]["solver_iterations"][: res.solves])
