"""Sweep knobs (env DREG_*) and print per-kernel CUDA-event times from tools/profile_step.py."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = sys.argv[1] if len(sys.argv) > 1 else "8"
combos = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{"DREG_TL": tl, "DREG_XVEC": v} for tl in (16, 32) for v in (2, 4)]
for c in combos:
    env = dict(os.environ, **{k: str(v) for k, v in c.items()})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profile_step.py"), B, "1"], env=env,
                         capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    print(json.dumps({"cfg": c, "res": line[0] if line else out.stderr[-300:]}), flush=True)
