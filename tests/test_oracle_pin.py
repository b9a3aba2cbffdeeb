"""Differential pin of the C restatement (oracle/dreg_oracle.c) against the UNMODIFIED
reference core compiled into oracle/_ref (oracle/Makefile `ref`): identical fp64
arithmetic, so every output must be bit-identical on randomised seeded inputs.
Also validates the oracle's FFT (oracle/fft_core.c, FFTW's stand-in) against numpy.
"""
import numpy as np
import pytest

from conftest import random_field, random_volume
from paper_2109_12688_b200 import abi, synth


@pytest.mark.parametrize("shape", [(4, 6, 5), (7, 3, 9), (16, 16, 16), (12, 10, 30)])
@pytest.mark.parametrize("n", [1, 2, 3])
def test_w_update_bit_exact(oracle, reference, shape, n):
    v, b = random_field(shape, 7 + n, 1.0), random_field(shape, 17 + n, 1.0)
    cfg = abi.solver_cfg(order=n, lambda_=1.5, theta=0.2)
    assert np.array_equal(oracle.w_update(v, b, cfg), reference.w_update(v, b, cfg))


@pytest.mark.parametrize("dt", [1, 2])
def test_solve_and_register_bit_exact(oracle, reference, dt):
    f, m = synth.make_pair(1, 31, (12, 16, 20))
    s = abi.solver_cfg(data_term=dt, order=2, lambda_=0.2, theta=0.5, max_iters=15, log_objective=True)
    vo, do = oracle.solve_velocity(f, m, s)
    vr, dr = reference.solve_velocity(f, m, s)
    assert np.array_equal(vo, vr)
    assert np.array_equal(do["objective"], dr["objective"])
    assert np.array_equal(do["constraint_residual"], dr["constraint_residual"])
    rc = abi.reg_cfg(abi.solver_cfg(data_term=dt, order=2, lambda_=0.2, theta=0.5, max_iters=15,
                                    log_objective=False), 1, (4,), (15,))
    po, wo, ro = oracle.register_pair(f, m, rc)
    pr, wr, rr = reference.register_pair(f, m, rc)
    assert np.array_equal(po, pr) and np.array_equal(wo, wr)
    assert ro.velocity_count == rr.velocity_count
    assert abi.level_logs(ro) == abi.level_logs(rr)


def test_pyramid_bit_exact(oracle, reference):
    f, m = synth.make_pair(1, 32, (16, 16, 16))
    s = abi.solver_cfg(data_term=1, order=2, lambda_=5.0, theta=0.05, log_objective=False)
    for prof in (abi.DREG_PROFILE_CAPPED, abi.DREG_PROFILE_CONVERGED):
        cfg = reference.make_registration_config(prof, s, 2)
        cfg.max_warps_per_level[0] = min(cfg.max_warps_per_level[0], 4)
        cfg.max_warps_per_level[1] = min(cfg.max_warps_per_level[1], 3)
        po, wo, ro = oracle.register_pair(f, m, cfg)
        pr, wr, rr = reference.register_pair(f, m, cfg)
        assert np.array_equal(po, pr) and np.array_equal(wo, wr)
        assert abi.level_logs(ro) == abi.level_logs(rr)


def test_field_ops_bit_exact(oracle, reference):
    shape = (9, 11, 10)
    img, d = random_volume(shape, 41), random_field(shape, 42, 2.0)
    for name in ["warp_image", "compose_deformation"]:
        a = getattr(oracle, name)(img if name == "warp_image" else d * np.float32(0.5), d)
        b = getattr(reference, name)(img if name == "warp_image" else d * np.float32(0.5), d)
        assert np.array_equal(a, b), name
    assert np.array_equal(oracle.image_gradient(img), reference.image_gradient(img))
    assert np.array_equal(oracle.jacobian_determinant(d * np.float32(0.4)), reference.jacobian_determinant(d * np.float32(0.4)))
    so, sr = oracle.jacobian_stats(d), reference.jacobian_stats(d)
    assert (so.nonpositive, so.interior, so.min_det) == (sr.nonpositive, sr.interior, sr.min_det)
    assert abs(so.pct_nonpositive - sr.pct_nonpositive) <= 1e-12
    assert np.array_equal(oracle.binomial_smooth(img), reference.binomial_smooth(img))
    assert np.array_equal(oracle.downsample(img), reference.downsample(img))


def test_errors_match(oracle, reference):
    f = random_volume((8, 8, 8), 3)
    m = f.copy()
    m[0, 0, 0] = np.inf
    cfg = abi.reg_cfg(abi.solver_cfg(max_iters=2), 1, (1,), (2,))
    for lib in (oracle, reference):
        with pytest.raises(Exception) as e:
            lib.register_pair(f, m, cfg)
        assert e.value.status == abi.DREG_NUMERIC
    small = random_volume((4, 4, 4), 3)
    cfg3 = reference.make_registration_config(abi.DREG_PROFILE_CAPPED, abi.solver_cfg(), 3)
    for lib in (oracle, reference):
        with pytest.raises(Exception) as e:
            lib.register_pair(small, small, cfg3)
        assert e.value.status == abi.DREG_INVALID_ARGUMENT


@pytest.mark.parametrize("shape", [(4, 4, 4), (5, 6, 7), (8, 16, 32), (3, 10, 9), (2, 2, 11)])
def test_oracle_fft_against_numpy(oracle, shape):
    """fft_core.c is FFTW's stand-in: check r2c/c2r via the w-update's lambda->0 and
    a direct spectral filter computed with numpy (pocketfft)."""
    v = random_field(shape, 5, 1.0)
    b = np.zeros_like(v)
    cfg = abi.solver_cfg(order=1, lambda_=0.7, theta=0.3)
    out = oracle.w_update(v, b, cfg)
    K = oracle.laplacian_symbol(1, abi.dims3(v))
    hx = shape[2] // 2 + 1
    ref = np.stack([np.fft.irfftn(np.fft.rfftn(v[..., c].astype(np.float64)) * (0.3 / (0.7 * K[:, :, :hx] + 0.3)),
                                  s=shape, axes=(0, 1, 2)) for c in range(3)], -1)
    assert np.abs(out - ref).max() <= 1e-6


def test_mkl_timing_build_matches_parity_build(reference):
    """The CPU-timing build of the reference (same objects, FFTW API over MKL DFTI,
    bench.py's cpu_baseline / --impl reference) computes the same registration as the
    parity build up to FFT rounding."""
    from oracle.oracle import CpuLib, available

    if not available("reference_mkl"):
        pytest.skip("oracle/_ref/libdreg_ref_mkl.so not built")
    mkl = CpuLib("reference_mkl")
    f, m = synth.make_pair(1, 5, (16, 32, 32))
    cfg = abi.reg_cfg(abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=50),
                      max_warps=(3,), max_admm_iters=(50,))
    p1, w1, r1 = reference.register_pair(f, m, cfg)
    p2, w2, r2 = mkl.register_pair(f, m, cfg)
    assert r1.velocity_count == r2.velocity_count
    assert np.max(np.abs(p1 - p2)) < 1e-5
    assert np.linalg.norm(p1 - p2) <= 1e-6 * np.linalg.norm(p1)


def _points(shape, seed, n=500):
    """sample points inside, on and outside the grid (clamp rule, volume.cpp:36-41)"""
    z, y, x = shape
    rng = np.random.default_rng(seed)
    p = rng.uniform(-2.0, [x + 1.0, y + 1.0, z + 1.0], (n, 3))
    p[:8] = [[0, 0, 0], [x - 1, y - 1, z - 1], [0.5, 0.5, 0.5], [x - 1.25, 0, 0], [-1, -1, -1],
             [x + 3, y + 3, z + 3], [1, 2, 3], [2.5, 0.0, 1.0]]
    return p


def test_trilinear_sample_bit_exact(oracle, reference):
    """volume.hpp:107,110: scalar and vector trilinear_sample, restatement vs reference."""
    shape = (7, 9, 8)
    img, fld = random_volume(shape, 61), random_field(shape, 62, 2.0)
    pts = _points(shape, 63)
    assert np.array_equal(oracle.trilinear_sample(img, pts), reference.trilinear_sample(img, pts))
    assert np.array_equal(oracle.trilinear_sample(fld, pts), reference.trilinear_sample(fld, pts))


@pytest.mark.parametrize("s", [1, 2])
def test_data_term_value_bit_exact(oracle, reference, s):
    shape = (6, 8, 10)
    t, w = random_volume(shape, 64), random_volume(shape, 65)
    g, v = random_field(shape, 66, 1.0), random_field(shape, 67, 0.5)
    assert oracle.data_term_value(t, w, g, v, s) == reference.data_term_value(t, w, g, v, s)
