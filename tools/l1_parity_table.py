"""Per-case l1 parity table: acceptance criterion 5's 13 registrations
(acceptance_main.cpp:261-291: translate (3,0,0), sphere -> ellipsoid, random smooth
seeds 3 and 100..109 at 32^3; l1, n 2, lambda 10, theta 0.05, capped, 3 levels) plus
the test_registration.cpp sphere / translate cases, GPU vs the oracle (bit-exact
restatement of the reference).  For each case: phi max-abs / rel-L2 for the default
policy (l1 -> fp64 point-wise + precise spectral) and for forced fp32 spectral
arithmetic, velocity counts, the oracle's own response to rounding-level
perturbations of the target (1 ulp and 1e-6 relative, two draws each: the
conditioning yardstick), and the unmodified reference linked against a different FFT
(MKL DFTI instead of the portable FFTW stand-in) -- the spread the reference itself
shows between two correct FFT libraries.  Prints a markdown table and writes JSON.

Usage (GPU box): python tools/l1_parity_table.py [--out gpurun_out/l1_parity.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, dreg  # noqa: E402


def capped(data_term, lam, levels, theta=0.05):
    s = abi.solver_cfg(data_term=data_term, order=2, lambda_=lam, theta=theta, log_objective=False)
    return dreg.make_registration_config(abi.DREG_PROFILE_CAPPED, s, levels)


def perturbed(img, seed=0, amp=6e-8):
    rng = np.random.default_rng(seed)
    return (img * (1.0 + rng.uniform(-1.0, 1.0, img.shape) * amp)).astype(np.float32)


def err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max()), float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "l1_parity.json"))
    a = ap.parse_args()
    ref = CpuLib("reference")
    ora = CpuLib("oracle")
    mkl = CpuLib("reference_mkl")  # the unmodified reference over a different (MKL) FFT
    cases = [("translate", dict(shift=(3.0, 0.0, 0.0)), (32, 32, 32), capped(1, 10.0, 3), "crit5"),
             ("sphere_ellipsoid", {}, (32, 32, 32), capped(1, 10.0, 3), "crit5")]
    cases += [("random_smooth", dict(seed=sd), (32, 32, 32), capped(1, 10.0, 3), "crit5") for sd in [3] + list(range(100, 110))]
    cases += [("sphere_ellipsoid", {}, (32, 32, 32), capped(1, 5.0, 3), "test_registration:247"),
              ("translate", dict(shift=(2.0, 0.0, 0.0)), (32, 32, 32), capped(1, 10.0, 3), "test_registration:217"),
              ("sphere_ellipsoid", {}, (32, 32, 32), capped(2, 10.0, 3), "l2 control")]
    rows = []
    with dreg.Context(0) as ctx:
        for kind, kw, shape, cfg, tag in cases:
            t, s, _, _ = ref.make_case(kind, shape, **kw)
            po, _, ro = ora.register_pair(t, s, cfg)
            ctx.set_precision(0)
            pg, _, rg = ctx.register_pair(t, s, cfg)
            ctx.set_precision(1)
            pf, _, rf = ctx.register_pair(t, s, cfg)
            ctx.set_precision(0)
            ulp = (0.0, 0.0)
            for amp in (6e-8, 1e-6):
                for sd in (0, 1):
                    pp, _, _ = ora.register_pair(perturbed(t, sd, amp), s, cfg)
                    e = err(pp, po)
                    ulp = (max(ulp[0], e[0]), max(ulp[1], e[1]))
            pm, _, rm = mkl.register_pair(t, s, cfg)
            row = dict(case=f"{kind} {kw}" if kw else kind, tag=tag, data_term=cfg.solver.data_term,
                       vc_oracle=ro.velocity_count, vc_gpu=rg.velocity_count, vc_gpu_fast=rf.velocity_count,
                       gpu=err(pg, po), gpu_fast=err(pf, po), oracle_1ulp=ulp, ref_mkl=err(pm, po),
                       vc_mkl=rm.velocity_count,
                       folding_gpu=int(ctx.jacobian_stats(pg).nonpositive))
            rows.append(row)
            print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)
    print("\n| case | criterion | velocity count oracle / GPU | GPU max-abs | GPU rel-L2 | fp32-spectral max-abs | "
          "fp32-spectral rel-L2 | oracle perturbed max-abs | oracle perturbed rel-L2 | reference (MKL FFT) max-abs | "
          "reference (MKL FFT) rel-L2 |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['case']} | {r['tag']} | {r['vc_oracle']} / {r['vc_gpu']} | {r['gpu'][0]:.2e} | {r['gpu'][1]:.2e} | "
              f"{r['gpu_fast'][0]:.2e} | {r['gpu_fast'][1]:.2e} | {r['oracle_1ulp'][0]:.2e} | {r['oracle_1ulp'][1]:.2e} | "
              f"{r['ref_mkl'][0]:.2e} | {r['ref_mkl'][1]:.2e} |")


if __name__ == "__main__":
    main()
