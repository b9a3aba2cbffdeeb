"""CPU model of the device FFT scheme (csrc/fft_device.cuh + the x-pass/plane kernels):
DIF forward stages leave digit-reversed order, the adjoint stages consume it, the
regulariser multiply is applied through position->frequency tables, and the x axis
uses the half-length r2c/c2r trick.  Checked against numpy.fft so index bugs surface
without a GPU.  The plan logic mirrors engine.cu make_plan / freq_of_pos.
"""
import numpy as np
import pytest


def make_plan(n):
    radix, rem = [], n
    while rem > 1:
        for r in (8, 4, 2, 3, 5, 7):
            if rem % r == 0:
                break
        else:
            r = 11
            while rem % r:
                r += 2
        radix.append(r)
        rem //= r
    n1, tws, ns = [], [], n
    for r in radix:
        n1.append(ns // r)
        tws.append(n // ns)
        ns //= r
    return radix, n1, tws


def freq_of_pos(plan, pos):
    radix, n1, _ = plan
    f, mult, p = 0, 1, pos
    for r, m in zip(radix, n1):
        k2 = p // m
        p -= k2 * m
        f += mult * k2
        mult *= r
    return f


def fft_lines(buf, n, inverse):
    """buf: (lines, n) complex, transformed in place along axis 1 (device stage loop)."""
    plan = make_plan(n)
    radix, n1s, twss = plan
    tw = np.exp(-2j * np.pi * np.arange(n) / n)
    order = range(len(radix) - 1, -1, -1) if inverse else range(len(radix))
    for s in order:
        r, n1, tws = radix[s], n1s[s], twss[s]
        ns = n1 * r
        W = np.exp(-2j * np.pi * np.outer(np.arange(r), np.arange(r)) / r)  # W[t,k]
        for b in range(n // r):
            blk, j1 = divmod(b, n1)
            idx = blk * ns + j1 + n1 * np.arange(r)
            x = buf[:, idx]
            t = tw[(j1 * np.arange(r) * tws)]
            if inverse:
                y = (x * np.conj(t)) @ np.conj(W)
            else:
                y = (x @ W) * t
            buf[:, idx] = y
    return plan


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 12, 16, 30, 64, 96, 128, 192, 22])
def test_dif_then_adjoint_roundtrip_and_order(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))
    b = x.copy()
    plan = fft_lines(b, n, inverse=False)
    pos_freq = np.array([freq_of_pos(plan, p) for p in range(n)])
    ref = np.fft.fft(x, axis=1)
    assert np.allclose(b, ref[:, pos_freq], atol=1e-9 * n)
    fft_lines(b, n, inverse=True)
    assert np.allclose(b / n, x, atol=1e-12 * n)


def r2c_half(line, M):
    L = M // 2
    z = (line[0::2] + 1j * line[1::2])[None, :].astype(complex)
    plan = fft_lines(z, L, inverse=False)
    pos = np.zeros(L, int)
    for p in range(L):
        pos[freq_of_pos(plan, p)] = p
    xtw = np.exp(-2j * np.pi * np.arange(L + 1) / M)
    X = np.zeros(L + 1, complex)
    for k in range(L + 1):
        zk = z[0, pos[k % L]]
        zc = np.conj(z[0, pos[(L - k) % L]])
        e = 0.5 * (zk + zc)
        o = 0.5 * (zk - zc) / 1j
        X[k] = e + xtw[k] * o
    return X


def c2r_half(X, M):
    L = M // 2
    plan = make_plan(L)
    pos = np.zeros(L, int)
    for p in range(L):
        pos[freq_of_pos(plan, p)] = p
    xtw = np.exp(-2j * np.pi * np.arange(L + 1) / M)
    X = X.copy()
    X[0] = X[0].real
    X[L] = X[L].real
    buf = np.zeros((1, L), complex)
    for k in range(L):
        A, B = X[k], np.conj(X[L - k])
        e, o = A + B, (A - B) * np.conj(xtw[k])
        buf[0, pos[k]] = e + 1j * o
    fft_lines(buf, L, inverse=True)
    out = np.zeros(M)
    out[0::2] = buf[0].real
    out[1::2] = buf[0].imag
    return out


@pytest.mark.parametrize("M", [2, 4, 6, 8, 10, 16, 64, 128, 256])
def test_half_length_r2c_c2r(M):
    rng = np.random.default_rng(M)
    x = rng.standard_normal(M)
    X = r2c_half(x, M)
    assert np.allclose(X, np.fft.rfft(x), atol=1e-9 * M)
    assert np.allclose(c2r_half(X, M) / M, x, atol=1e-12 * M)


@pytest.mark.parametrize("shape", [(4, 6, 8), (5, 4, 4), (8, 16, 12)])
def test_plane_multiply_through_position_tables(shape):
    """y/z DIF, multiply by m(q_true, r_true), adjoint == numpy filter on the plane."""
    Nz, Ny = shape[0], shape[1]
    rng = np.random.default_rng(1)
    plane = rng.standard_normal((Nz, Ny)) + 1j * rng.standard_normal((Nz, Ny))
    mq = rng.random(Ny)
    mr = rng.random(Nz)
    b = plane.copy()
    py = fft_lines(b, Ny, False)            # rows (y lines)
    bt = np.ascontiguousarray(b.T)
    pz = fft_lines(bt, Nz, False)           # columns (z lines)
    fy = np.array([freq_of_pos(py, p) for p in range(Ny)])
    fz = np.array([freq_of_pos(pz, p) for p in range(Nz)])
    bt *= (mq[fy][:, None] + mr[fz][None, :])
    fft_lines(bt, Nz, True)
    b = bt.T.copy()
    fft_lines(b, Ny, True)
    ref = np.fft.ifft2(np.fft.fft2(plane) * (mr[:, None] + mq[None, :]))
    assert np.allclose(b / (Ny * Nz), ref, atol=1e-10)
