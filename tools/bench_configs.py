"""Per-config registration timing on one GPU (BASELINE.json configs 1, 2 (n=1,2,3), 4, 5).

    python tools/bench_configs.py [reps]

Each config: one seeded pair (its own phantom) registered with its solver settings
(SURVEY.md §8(d), D1-D4), inputs resident on the device, CUDA-event timed after a
warm-up; prints one JSON line per config with ms per registration, the number of
velocity fields / iterations run and the folding count.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_12688_b200 import dreg, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = dreg.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
runs = [("config1", None), ("config2", 1), ("config2", 2), ("config2", 3), ("config4", None), ("config5", None)]
for name, order in runs:
    c = synth.CONFIGS[name]
    f, m = synth.make_pair(c["synth"], c["seed"], c["shape"])
    N = f.size
    t = torch.from_numpy(f.reshape(1, N)).cuda()
    s = torch.from_numpy(m.reshape(1, N)).cuda()
    phi = torch.empty((1, 3, N), device="cuda")
    cfg = synth.config_cfg(name, order=order)
    dims = c["shape"][::-1]
    res = ctx.register_batch_device(1, t.data_ptr(), s.data_ptr(), dims, cfg, phi.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        res = ctx.register_batch_device(1, t.data_ptr(), s.data_ptr(), dims, cfg, phi.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    js = ctx.jacobian_stats_device(phi[0].data_ptr(), dims)
    r = res[0]
    print(json.dumps({"config": name, "order": order or c["order"], "shape_zyx": c["shape"], "ms_per_registration": ms,
                      "velocity_count": r.velocity_count, "solves": r.solves,
                      "iterations_per_solve": c["iters"], "folding_voxels": int(js.nonpositive),
                      "min_det": js.min_det}), flush=True)
