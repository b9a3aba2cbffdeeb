"""Memory-safety and race evidence without compute-sanitizer (closed on the GPU pool:
runs under it left GPUs needing a reset -- see profiles/r2_sanitizer.md).

* Guard bands (DREG_GUARD=1): every device buffer is allocated with 64 KB of a fixed
  byte pattern on each side; after each registration / solve the library verifies all
  of them and fails the call if any kernel wrote past either end of any buffer.
* Scheduling-invariance: shared-memory or cross-CTA races show up as run-to-run or
  schedule-dependent bits.  The same registrations are repeated with graphs on / off,
  different launch chunkings and a capped persistent x-pass grid (DREG_XPASS_SMS), and
  every output field must be bit-identical (the reference's own invariant,
  acceptance_main.cpp:358-393)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.path.join(ROOT, "tools", "sanitize_run.py")


def _run(args, **env):
    e = dict(os.environ)
    e.update({k: str(v) for k, v in env.items()})
    p = subprocess.run([sys.executable, RUN, *args], capture_output=True, text=True, timeout=600, env=e, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    return [ln.split()[1] for ln in p.stdout.splitlines() if ln.startswith("digest")][0]


GRIDS = [["--shape", "16,32,32", "--data-term", "1"], ["--shape", "64,64,64"], ["--shape", "64,128,128"],
         ["--shape", "24,40,48", "--precise", "1", "--warps", "1", "--iters", "3"]]


@pytest.mark.parametrize("grid", GRIDS, ids=lambda g: g[1])
def test_guard_bands_intact(grid):
    plain = _run(grid)
    guarded = _run(grid, DREG_GUARD=1)
    assert guarded == plain  # guard mode changes nothing but the allocation layout


@pytest.mark.parametrize("grid", GRIDS[:3], ids=lambda g: g[1])
def test_schedule_invariance(grid):
    base = _run(grid + ["--pairs", "3"])
    assert _run(grid + ["--pairs", "3"]) == base  # run to run
    assert _run(grid + ["--pairs", "3", "--graphs", "1"]) == base
    assert _run(grid + ["--pairs", "3", "--chunk", "1"]) == base
    assert _run(grid + ["--pairs", "3", "--chunk", "2", "--graphs", "1"]) == base
    assert _run(grid + ["--pairs", "3"], DREG_XPASS_SMS=37) == base
