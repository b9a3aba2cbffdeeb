"""Timing of the spectral w-update: cuFFT (R2C -> multiplier -> C2R through torch.fft,
library code) against this repo's per-iteration kernels (fused x-pass + yz plane,
which also carry ALL the point-wise ADMM work), on batches of config-2-shaped pairs
(64x128x128, 3 components each).  CUDA events on the launching stream, 20 reps after
warm-up, L2 working set >> 126 MB.  Writes a markdown table to stdout.

Usage (GPU box): python tools/cufft_timing.py [--pairs 8 32 128]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_12688_b200 import abi, dreg, synth  # noqa: E402

SHAPE = (64, 128, 128)


def time_cuda(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, nargs="+", default=[8, 32, 128])
    a = ap.parse_args()
    z, y, x = SHAPE
    N = z * y * x
    K = dreg.laplacian_symbol(2, (x, y, z))[:, :, : x // 2 + 1]
    mult = torch.as_tensor(1.0 / (0.1 * K + 1.0) / N, device="cuda", dtype=torch.float32)
    cfg = synth.config_cfg("config3")
    print("| pairs | cuFFT R2C+mult+C2R ms | cuFFT us / pair-iter | ours x-pass+plane ms | ours us / pair-iter | ours / cuFFT |")
    print("|---|---|---|---|---|---|")
    for P in a.pairs:
        u = torch.randn((P * 3, z, y, x), device="cuda", dtype=torch.float32)
        spec = torch.empty((P * 3, z, y, x // 2 + 1), device="cuda", dtype=torch.complex64)
        out = torch.empty_like(u)

        def cufft():
            torch.fft.rfftn(u, dim=(1, 2, 3), out=spec)
            spec.mul_(mult)
            torch.fft.irfftn(spec, s=(z, y, x), dim=(1, 2, 3), norm="forward", out=out)

        t_cu = time_cuda(cufft)
        del u, spec, out
        torch.cuda.empty_cache()
        F, M = synth.make_batch(3, 1000, P, SHAPE)
        tgt = torch.from_numpy(F.reshape(P, N)).cuda()
        src = torch.from_numpy(M.reshape(P, N)).cuda()
        with dreg.Context(0) as ctx:
            ctx.set_stream(torch.cuda.current_stream().cuda_stream)
            ctx.register_batch_device(P, tgt.data_ptr(), src.data_ptr(), SHAPE[::-1], cfg)
            tk = ctx.time_kernels(20, cfg.solver)
        ours = tk["xpass_ms"] + tk["plane_ms"]
        print(f"| {P} | {t_cu:.3f} | {1e3 * t_cu / P:.1f} | {ours:.3f} | {1e3 * ours / P:.1f} | {ours / t_cu:.2f} |",
              flush=True)
        del tgt, src
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
