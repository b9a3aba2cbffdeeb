"""Run the CPU oracle (bit-exact with the reference) on all 256 config-3 pairs and
record per-pair results in tests/golden/config3_oracle.json: velocity_count, number of
solve_velocity calls, the mean-SAD log, the interior folding count / min det J, and
phi digests (sum, sum of squares, max |phi|) for parity checks of the GPU batch path.

    python tools/run_config3_oracle.py [threads]
"""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.oracle import CpuLib  # noqa: E402
from paper_2109_12688_b200 import abi, synth  # noqa: E402

threads = int(sys.argv[1]) if len(sys.argv) > 1 else 6
out_path = os.path.join(ROOT, "tests", "golden", "config3_oracle.json")
results = {}
if os.path.exists(out_path):
    results = json.load(open(out_path))["pairs"]
lock = threading.Lock()
todo = [s for s in range(1000, 1256) if str(s) not in results]
cfg = synth.config_cfg("config3")


def worker():
    lib = CpuLib("oracle")
    while True:
        with lock:
            if not todo:
                return
            seed = todo.pop(0)
        f, m = synth.make_pair(3, seed, (64, 128, 128))
        t0 = time.time()
        phi, warped, res = lib.register_pair(f, m, cfg)
        js = lib.jacobian_stats(phi)
        lg = abi.level_logs(res)[0]
        rec = {
            "velocity_count": res.velocity_count,
            "solves": res.solves,
            "mean_sad": lg["mean_sad"],
            "solver_iterations": lg["solver_iterations"],
            "folding": int(js.nonpositive),
            "min_det": js.min_det,
            "phi_sum": float(phi.astype(np.float64).sum()),
            "phi_sumsq": float((phi.astype(np.float64) ** 2).sum()),
            "phi_maxabs": float(np.abs(phi).max()),
            "seconds": time.time() - t0,
        }
        with lock:
            results[str(seed)] = rec
            json.dump({"config": "config3 (config-2 solver, n=2, 7 x 50, levels 1)", "pairs": results},
                      open(out_path, "w"), indent=0)
            print(seed, rec["velocity_count"], rec["solves"], f"{rec['seconds']:.1f}s", flush=True)


ts = [threading.Thread(target=worker) for _ in range(threads)]
for t in ts:
    t.start()
for t in ts:
    t.join()
