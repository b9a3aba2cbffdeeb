"""Small registration workload for compute-sanitizer (tools/sanitize.sh).

Registers `--pairs` seeded config-3 phantoms at `--shape` (numpy z,y,x) with the
config-2 solver for `--warps` fields x `--iters` iterations (graphs off by default so
each kernel is a separate launch), then prints a SHA-256 digest of every output field:
tests/test_guard.py runs it under DREG_GUARD=1 (guard bands around every device
buffer) and under scheduling variations (chunking, graphs, x-pass CTA count) that must
not change a single bit.  Covers, at M = 64/128 with
Ny, Nz in {64, 128}: xpass_fast_kernel (k = 0, 1), xpass_pipe_kernel (k >= 2),
plane_reg_kernel, grad_diff, compose_decide, prep/level/finalize; at 16x32x32 the
generic x-pass and plane_fast_kernel.  Also one solve_velocity with the objective
logged (X_FWD / energy plane) and one Jacobian.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2109_12688_b200 import abi, dreg, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="64,64,64")
    ap.add_argument("--pairs", type=int, default=2)
    ap.add_argument("--warps", type=int, default=2)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--data-term", type=int, default=2)
    ap.add_argument("--precise", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--graphs", type=int, default=0)
    a = ap.parse_args()
    shape = tuple(int(s) for s in a.shape.split(","))
    F, M = synth.make_batch(3, 1000, a.pairs, shape)
    s = abi.solver_cfg(data_term=a.data_term, order=2, lambda_=0.1, theta=1.0, max_iters=a.iters,
                       log_objective=False)
    cfg = abi.reg_cfg(s, levels=1, max_warps=(a.warps,), max_admm_iters=(a.iters,))
    with dreg.Context(0) as ctx:
        ctx.set_use_graphs(bool(a.graphs))
        ctx.set_batch_chunk(a.chunk)
        ctx.set_precision(2 if a.precise else 1)
        phis, warped, res = ctx.register_batch(list(F), list(M), cfg)
        js = ctx.jacobian_stats(phis[0])
        s2 = abi.solver_cfg(data_term=a.data_term, order=2, lambda_=0.1, theta=1.0, max_iters=3,
                            log_objective=True)
        v, diag = ctx.solve_velocity(F[0], M[0], s2)
    import hashlib

    h = hashlib.sha256()
    for p in phis:
        h.update(np.ascontiguousarray(p).tobytes())
    h.update(np.ascontiguousarray(v).tobytes())
    print("ok", shape, [r.velocity_count for r in res], js.nonpositive, float(np.abs(v).max()))
    print("digest", h.hexdigest())


if __name__ == "__main__":
    main()
