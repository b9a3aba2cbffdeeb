"""CPU model of the spectral-state ADMM iteration (plane_fast.cuh MODE 2 + X_SS).

The product carries the accelerated-ADMM state of admm.cpp:275-308 as two Fourier-domain
iterates U_j, U_{j-1} (w = m U, b = (1 - m) U, extrapolation linear).  This test restates that
recurrence in numpy (fp64 and fp32) and checks it against the CPU oracle's solve_velocity --
the algebra the CUDA kernels rely on, without a GPU."""
import numpy as np
import pytest

from oracle.oracle import CpuLib
from paper_2109_12688_b200 import abi, synth


def _coefs(n):
    a, out = 1.0, []
    for _ in range(n):
        an = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * a * a))
        out.append((a - 1.0) / an)
        a = an
    return out


def _spectral_state_solve(f, m, g, K, lam, theta, iters, real, cplx):
    """v after `iters` iterations; `real` / `cplx` are the working dtypes."""
    shape = f.shape
    d = (m.astype(np.float64) - f.astype(np.float64)).astype(real)
    gx = [g[..., i].astype(real) for i in range(3)]
    gg = gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2]
    one_m = (lam * K / (lam * K + theta)).astype(real)          # 1 - m
    two_m1 = ((theta - lam * K) / (lam * K + theta)).astype(real)  # 2 m - 1
    th = real(theta)
    c = _coefs(iters)
    hx = shape[2] // 2 + 1
    zero = np.zeros((shape[0], shape[1], hx), cplx)
    Z, U1, U0, Ut = ([zero.copy() for _ in range(3)] for _ in range(4))
    v = None
    for k in range(iters):
        z = [np.fft.irfftn(Z[i], s=shape, axes=(0, 1, 2)).astype(real) for i in range(3)]
        s = (gx[0] * z[0] + gx[1] * z[1] + gx[2] * z[2] + d) / (th + gg)   # admm.cpp:41-63 (l2)
        v = [(z[i] - gx[i] * s).astype(real) for i in range(3)]
        ck = real(c[k])
        for i in range(3):
            Un = (np.fft.rfftn(v[i], axes=(0, 1, 2)).astype(cplx) + one_m * Ut[i]).astype(cplx)
            U0[i], U1[i] = U1[i], Un
            Ut[i] = (U1[i] + ck * (U1[i] - U0[i])).astype(cplx)   # admm.cpp:130-139 on w and b at once
            Z[i] = (two_m1 * Ut[i]).astype(cplx)
    return np.stack(v, -1)


@pytest.mark.parametrize("order", [1, 2, 3])
def test_spectral_state_recurrence_equals_reference_solve(order):
    shape, iters, lam, theta = (12, 16, 20), 30, 0.1, 1.0
    ora = CpuLib("oracle")
    f, m = synth.make_pair(2, 3, shape)
    f, m = ora.normalize_intensity_pair(f, m)
    cfg = abi.solver_cfg(data_term=2, order=order, lambda_=lam, theta=theta, max_iters=iters, tol=0.0,
                         log_objective=False)
    v_ref, info = ora.solve_velocity(f, m, cfg)
    assert info["iterations"] == iters
    g = ora.image_gradient(m)
    K = np.asarray(ora.laplacian_symbol(order, shape[::-1]), np.float64).reshape(shape)[..., : shape[2] // 2 + 1]
    scale = float(np.abs(v_ref).max())
    # fp64: the reformulation is the same recurrence (differences = the reference's fp32 field rounding)
    v64 = _spectral_state_solve(f, m, g, K, lam, theta, iters, np.float64, np.complex128)
    assert np.abs(v64 - v_ref).max() <= 2e-5 * max(scale, 1.0)
    # fp32: what the kernels compute; inside the parity contract with room to spare
    v32 = _spectral_state_solve(f, m, g, K, lam, theta, iters, np.float32, np.complex64)
    err = v32.astype(np.float64) - v_ref
    assert np.abs(err).max() <= 2e-4 * max(scale, 1.0)
    assert np.linalg.norm(err) <= 1e-4 * np.linalg.norm(v_ref)
