"""Time the host-buffer registration path (dreg_cuda_register_batch, pinned buffers) for
a few batch-chunk settings:  python tools/e2e_probe.py [pairs] [reps]"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2109_12688_b200 import abi, dreg, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
SHAPE = (64, 128, 128)
F, M = synth.make_batch(3, 1000, B, SHAPE)
cfg = synth.config_cfg("config3")
hT, hS = torch.from_numpy(F).pin_memory(), torch.from_numpy(M).pin_memory()
hP = torch.empty((B, *SHAPE, 3), dtype=torch.float32).pin_memory()
hW = torch.empty((B, *SHAPE), dtype=torch.float32).pin_memory()
Fp = C.POINTER(C.c_float)
arr = lambda t: (Fp * B)(*[C.cast(t[i].data_ptr(), Fp) for i in range(B)])  # noqa: E731
Ta, Sa, Pa, Wa = arr(hT), arr(hS), arr(hP), arr(hW)
resb = (abi.PairResult * B)()
with dreg.Context(0) as ctx:
    def run():
        ctx._check(ctx.lib.dreg_cuda_register_batch(ctx.h, B, Ta, Sa, abi.dims3(SHAPE[::-1]), abi.Spacing3(1, 1, 1),
                                                    C.byref(cfg), Pa, Wa, resb))
    dev = torch.zeros(B, *SHAPE, device="cuda")
    for chunk in [0, B // 2, B // 4]:
        ctx.set_batch_chunk(chunk)
        run()
        ts = []
        for _ in range(R):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run()
            ts.append(time.perf_counter() - t0)
        print(f"chunk {chunk}: " + " ".join(f"{B / t:.1f}" for t in ts) + " reg/s", flush=True)
