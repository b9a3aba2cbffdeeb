"""bench.py's multi-GPU launcher (BASELINE config 3): `--gpus N` outside
torchrun re-launches N ranks; config 3's 256 pairs are split 256/N per rank with
disjoint seeds (strong scaling), or N x --pairs with --weak; a box with fewer than N
GPUs is refused instead of being reported as an N-GPU run.  CPU only (gloo dry run)."""
import json
import os
import subprocess
import sys

import pytest

from paper_2109_12688_b200 import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=240):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""  # the refusal test must see zero devices even on a GPU box
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


def _json_line(out: str) -> dict:
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("gpus", [2, 4])
def test_dry_run_strong_split(gpus):
    p = _run("--gpus", str(gpus), "--dry-run")
    assert p.returncode == 0, p.stderr[-2000:]
    j = _json_line(p.stdout)
    assert j["n_gpus"] == gpus and j["scaling"] == "strong" and j["disjoint"]
    assert j["pairs_total"] == 256
    per = 256 // gpus
    for r in range(gpus):
        assert j["seeds_by_rank"][str(r)] == [1000 + r * per, 1000 + (r + 1) * per - 1, per]
    assert j["max_over_ranks"] == gpus - 1


def test_dry_run_weak():
    p = _run("--gpus", "2", "--dry-run", "--weak", "--pairs", "8")
    assert p.returncode == 0, p.stderr[-2000:]
    j = _json_line(p.stdout)
    assert j["scaling"] == "weak" and j["pairs_total"] == 16 and j["disjoint"]


def test_refuses_missing_gpus():
    p = _run("--gpus", "2", "--steps", "1", "--warmup", "1")
    assert p.returncode == 2
    assert "only 0 CUDA device" in p.stderr


def test_split_pairs_uneven():
    blocks = [shard.split_pairs(r, 3, 256) for r in range(3)]
    assert [len(b) for b in blocks] == [85, 85, 86]
    assert sum(blocks, []) == list(range(1000, 1256))
    assert shard.rank_seeds(1, 8, 256, weak=False) == list(range(1032, 1064))
    assert shard.rank_seeds(1, 2, 4, weak=True) == [1004, 1005, 1006, 1007]
