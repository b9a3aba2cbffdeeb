"""Profiling driver: one batched registration (short) + per-kernel timing loop.

Used under ncu (launch list and --set full captures of xpass_kernel / plane_kernel).
  python tools/profile_step.py [pairs] [warps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2109_12688_b200 import abi, dreg, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
shape = (64, 128, 128)
F, M = synth.make_batch(3, 1000, B, shape)
cfg = synth.config_cfg("config3")
cfg.max_warps_per_level[0] = K
with dreg.Context(0) as ctx:
    if os.environ.get("DREG_CHUNK"):  # pairs per device launch (default: auto)
        ctx.set_batch_chunk(int(os.environ["DREG_CHUNK"]))
    phis, warps, res = ctx.register_batch(list(F), list(M), cfg, want_phi=False, want_warped=False)
    if os.environ.get("DREG_DBG_SKIP_TK"):  # timing-only knob for the kernel loop (not the registration)
        os.environ["DREG_DBG_SKIP"] = os.environ["DREG_DBG_SKIP_TK"]
    tk = ctx.time_kernels(5)
    print({k: (float(v) if not isinstance(v, int) else v) for k, v in tk.items()})
    print("launches", ctx.kernel_launches(), "velocity_counts", [r.velocity_count for r in res])
