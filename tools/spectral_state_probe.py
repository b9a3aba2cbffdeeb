"""CPU probe (no GPU): fp32 rounding behaviour of the spectral-state ADMM iteration.

The product's fused iteration keeps w_{k-1}, b_{k-1}, b_{k-2} as real-space fp32 fields.
The spectral-state form keeps U_k = FFT(v_k + b_hat_{k-1}) instead and uses
   w_k = m U_k,  b_k = (1 - m) U_k,  w_hat_k - b_hat_k = (2m - 1) Ut_k,  b_hat_k = (1 - m) Ut_k,
   Ut_k = U_k + c_{k-1} (U_k - U_{k-1})            (admm.cpp:66-101,130-153,275-308)
so an iteration is  z = IFFT((2m-1) Ut),  v = prox(z; g, d),  U' = FFT(v) + (1-m) Ut.
This script runs both forms in numpy fp32 (scipy pocketfft single precision) against the
CPU oracle's solve_velocity on a config-2 style pair and prints the velocity errors.

    python tools/spectral_state_probe.py [z y x] [iters] [order]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import scipy.fft as sf  # noqa: E402

from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, synth  # noqa: E402

shape = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (32, 64, 64)
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 50
order = int(sys.argv[5]) if len(sys.argv) > 5 else 2
lam, theta = 0.1, 1.0
ora = CpuLib("oracle")
f, m = synth.make_pair(2, 2, shape)
f, m = ora.normalize_intensity_pair(f, m)
f, m = ora.binomial_smooth(f), ora.binomial_smooth(m)
cfg = abi.solver_cfg(data_term=2, order=order, lambda_=lam, theta=theta, max_iters=iters, tol=0.0, log_objective=False)
v_ref, info = ora.solve_velocity(f, m, cfg)
g = ora.image_gradient(m)  # [z,y,x,3]
d = (m.astype(np.float64) - f.astype(np.float64)).astype(np.float32)
K = ora.laplacian_symbol(order, f.shape[::-1])  # [z,y,hx]?
K = np.asarray(K, np.float64).reshape(shape)[..., : shape[2] // 2 + 1]
F32, C64 = np.float32, np.complex64
mult = (theta / (lam * K + theta)).astype(F32)
one_m = (lam * K / (lam * K + theta)).astype(F32)
two_m1 = ((theta - lam * K) / (lam * K + theta)).astype(F32)


def coefs(n):
    a, out = 1.0, []
    for _ in range(n):
        an = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * a * a))
        out.append((a - 1.0) / an)
        a = an
    return out


c = coefs(iters)
assert abs(ora.nesterov_next_alpha(1.0) - 0.5 * (1 + np.sqrt(5.0))) < 1e-15
gx = [g[..., i].astype(F32) for i in range(3)]
gg = gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2]
th = F32(theta)


def prox(z):  # z: list of 3 fp32 arrays (w_hat - b_hat); pointwise.cuh v_update_voxel_f32 (l2)
    gu = gx[0] * z[0] + gx[1] * z[1] + gx[2] * z[2]
    s = (gu + d) / (th + gg)
    return [(z[i] - gx[i] * s).astype(F32) for i in range(3)]


def fwd(a):
    return sf.rfftn(a.astype(F32), axes=(0, 1, 2)).astype(C64)


def inv(A):
    return sf.irfftn(A.astype(C64), s=shape, axes=(0, 1, 2)).astype(F32)


def real_space():
    zero = [np.zeros(shape, F32) for _ in range(3)]
    wh, bh, wp, bp = zero, zero, zero, zero
    for k in range(iters):
        v = prox([wh[i] - bh[i] for i in range(3)])
        w = [inv(fwd(v[i] + bh[i]) * mult) for i in range(3)]
        b = [(bh[i] + (v[i] - w[i])).astype(F32) for i in range(3)]
        ck = F32(c[k])
        wh = [(w[i] + ck * (w[i] - wp[i])).astype(F32) for i in range(3)]
        bh = [(b[i] + ck * (b[i] - bp[i])).astype(F32) for i in range(3)]
        wp, bp = w, b
    return np.stack(v, -1)


def spectral_state():
    hx = shape[2] // 2 + 1
    Z = [np.zeros((shape[0], shape[1], hx), C64) for _ in range(3)]
    U1 = [z.copy() for z in Z]  # U_{k}
    U0 = [z.copy() for z in Z]  # U_{k-1}
    Ut = [z.copy() for z in Z]
    for k in range(iters):
        z = [inv(Z[i]) for i in range(3)]
        v = prox(z)
        ck = F32(c[k])
        for i in range(3):
            Un = (fwd(v[i]) + one_m * Ut[i]).astype(C64)
            U0[i], U1[i] = U1[i], Un
            Ut[i] = (U1[i] + ck * (U1[i] - U0[i])).astype(C64)
            Z[i] = (two_m1 * Ut[i]).astype(C64)
    return np.stack(v, -1)


def report(name, v):
    e = v.astype(np.float64) - v_ref.astype(np.float64)
    print(f"{name:16s} max-abs {np.abs(e).max():.3e}  rel-L2 {np.linalg.norm(e) / np.linalg.norm(v_ref):.3e}")


print(f"shape {shape} iters {iters} order {order}  |v_ref| max {np.abs(v_ref).max():.3f}")
va = real_space()
report("real-space fp32", va)
vb = spectral_state()
report("spectral fp32", vb)
e = va.astype(np.float64) - vb
print(f"between the two  max-abs {np.abs(e).max():.3e}")


def spectral_state_mixed():
    """fp32 transforms and v-update, fp64 state recurrence (U, Ut) -- what a mixed mode would do."""
    hx = shape[2] // 2 + 1
    C128 = np.complex128
    one_m64 = lam * K / (lam * K + theta)
    two_m164 = (theta - lam * K) / (lam * K + theta)
    Z = [np.zeros((shape[0], shape[1], hx), C64) for _ in range(3)]
    U1 = [np.zeros((shape[0], shape[1], hx), C128) for _ in range(3)]
    U0 = [z.copy() for z in U1]
    Ut = [z.copy() for z in U1]
    for k in range(iters):
        z = [inv(Z[i]) for i in range(3)]
        v = prox(z)
        for i in range(3):
            Un = fwd(v[i]).astype(C128) + one_m64 * Ut[i]
            U0[i], U1[i] = U1[i], Un
            Ut[i] = U1[i] + c[k] * (U1[i] - U0[i])
            Z[i] = (two_m164 * Ut[i]).astype(C64)
    return np.stack(v, -1)


if len(sys.argv) > 6:
    report("fp64 state mix", spectral_state_mixed())
