"""cuFFT cross-check of the hand-written spectral w-update (north_star: "cross-checked
against cuFFT").  The reference's w-update (admm.cpp:66-101) is, per component c,
w_c = IFFT(FFT(v_c + b_hat_c) * theta / (lambda K_n + theta) / N) with FFTW r2c/c2r
(fft.cpp:52-55,67-69).  Here the same operator is built from cuFFT R2C/C2R (through
torch.fft on the device -- library code, test only) and compared with
dreg_cuda_w_update (x r2c in the x-pass, y/z FFTs + multiplier in the plane kernel,
x c2r): cuFFT in fp64 is the yardstick; our fp32 path must sit within the reference's
own pin (1e-5 max|ref|, test_admm.cpp:184-211) and within a small factor of cuFFT's own
fp32 error.  tools/cufft_timing.py times the two paths (profiles/r2_cufft.md)."""
import numpy as np
import pytest

from conftest import random_field
from paper_2109_12688_b200 import abi, dreg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def cufft_w_update(v, bh, cfg, dtype):
    """w = C2R(R2C(v + b_hat) * theta / (lambda K_n + theta)); torch's irfftn divides by N."""
    z, y, x, _ = v.shape
    K = dreg.laplacian_symbol(cfg.order, (x, y, z))[:, :, : x // 2 + 1]  # Dims3 order in, (z, y, x) out
    mult = torch.as_tensor(cfg.theta / (cfg.lambda_ * K + cfg.theta), device="cuda", dtype=dtype)
    u = torch.as_tensor(v.astype(np.float64) + bh.astype(np.float64), device="cuda", dtype=dtype)
    u = u.permute(3, 0, 1, 2)  # [c][z][y][x]
    spec = torch.fft.rfftn(u, dim=(1, 2, 3))
    w = torch.fft.irfftn(spec * mult, s=(z, y, x), dim=(1, 2, 3))
    return w.permute(1, 2, 3, 0).cpu().numpy()


SHAPES = [(64, 128, 128), (32, 64, 64), (16, 32, 48), (12, 10, 6), (48, 96, 80), (24, 27, 40)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("order", [1, 2, 3])
def test_w_update_matches_cufft(ctx, shape, order):
    v = random_field(shape, 300 + order, 1.0)
    bh = random_field(shape, 400 + order, 1.0)
    cfg = abi.solver_cfg(order=order, lambda_=2.0, theta=0.1)
    ours = ctx.w_update(v, bh, cfg).astype(np.float64)
    ref64 = cufft_w_update(v, bh, cfg, torch.float64)
    cu32 = cufft_w_update(v, bh, cfg, torch.float32).astype(np.float64)
    scale = np.abs(ref64).max()
    e_ours = np.abs(ours - ref64).max()
    e_cu32 = np.abs(cu32 - ref64).max()
    print(f"{shape} n={order}: ours {e_ours / scale:.2e}, cuFFT fp32 {e_cu32 / scale:.2e} (x max|w|)")
    assert e_ours <= 1e-5 * scale
    assert e_ours <= max(4.0 * e_cu32, 1e-6 * scale)


def test_w_update_precise_matches_cufft_fp64(ctx):
    """fp64 butterflies (precise mode) against cuFFT fp64: only the final fp32 store
    differs, so the distance is a few fp32 ulps of the output."""
    shape = (32, 64, 64)
    v, bh = random_field(shape, 501, 1.0), random_field(shape, 502, 1.0)
    cfg = abi.solver_cfg(order=3, lambda_=0.05, theta=0.5, max_iters=200)
    ctx.set_precision(2)
    try:
        ours = ctx.w_update(v, bh, cfg).astype(np.float64)
    finally:
        ctx.set_precision(0)
    ref64 = cufft_w_update(v, bh, cfg, torch.float64)
    assert np.abs(ours - ref64).max() <= 2e-7 * np.abs(ref64).max()
