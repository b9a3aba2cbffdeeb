"""Multi-GPU batch through the C ABI (dreg_cuda_multi_*): contiguous
pair shards, one host thread + context per device, ONE NCCL all-gather of the
fixed-size per-pair records.  CPU tests pin the shard dealing and the gather layout
(the pure host helpers); the GPU test runs the whole path on the one device a gpurun
box has and checks every pair against the single-context batch bit for bit."""
import ctypes as C

import numpy as np
import pytest

from paper_2109_12688_b200 import abi, dreg, synth


def test_record_is_64_bytes():
    assert C.sizeof(abi.PairRecord) == 64


@pytest.mark.parametrize("n,shards", [(256, 1), (256, 2), (256, 8), (7, 3), (3, 8), (0, 2)])
def test_shard_range_covers_pairs_once(n, shards):
    got = [dreg.shard_range(n, shards, s) for s in range(shards)]
    assert got[0][0] == 0 and got[-1][1] == n
    for (b0, e0), (b1, e1) in zip(got, got[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in got]
    assert max(sizes) - min(sizes) <= 1
    if n == 256 and shards == 8:
        assert got[3] == (96, 128)
    with pytest.raises(ValueError):
        dreg.shard_range(n, shards, shards)


def _gathered(n, shards, cap):
    """The all-gather layout: shard s's records first, then padding (pair = -1)."""
    buf = (abi.PairRecord * (shards * cap))()
    for s in range(shards):
        b, e = dreg.shard_range(n, shards, s)
        for i in range(cap):
            r = buf[s * cap + i]
            if i < e - b:
                r.pair, r.device, r.velocity_count, r.final_mean_sad = b + i, s, 100 + b + i, 0.5 * (b + i)
            else:
                r.pair, r.device = -1, -1
    return buf


def test_records_unpack_pair_order():
    lib = dreg.load_library()
    n, shards, cap = 11, 3, 5
    buf = _gathered(n, shards, cap)
    out = (abi.PairRecord * n)()
    assert lib.dreg_records_unpack(buf, shards, cap, n, out) == abi.DREG_OK
    assert [r.pair for r in out] == list(range(n))
    assert [r.velocity_count for r in out] == [100 + i for i in range(n)]
    assert [r.device for r in out] == [0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2]


@pytest.mark.parametrize("corrupt", ["missing", "duplicate", "padding", "small_cap"])
def test_records_unpack_rejects_bad_layout(corrupt):
    lib = dreg.load_library()
    n, shards, cap = 11, 3, 5
    buf = _gathered(n, shards, cap)
    out = (abi.PairRecord * n)()
    if corrupt == "missing":
        buf[0].pair = -1
    elif corrupt == "duplicate":
        buf[1].pair = 0
    elif corrupt == "padding":
        buf[cap - 1].pair = 3  # shard 0 holds 3 pairs; slot 4 is padding
    else:
        cap = 3
    assert lib.dreg_records_unpack(buf, shards, cap, n, out) == abi.DREG_INVALID_ARGUMENT


@pytest.mark.gpu
def test_multi_one_device_matches_single_context(ctx):
    F, M = synth.make_batch(3, 1000, 5, (16, 32, 64))
    s = abi.solver_cfg(data_term=2, order=2, lambda_=0.1, theta=1.0, max_iters=20, log_objective=False)
    cfg = abi.reg_cfg(s, 1, (3,), (20,))
    phis, warps, res = ctx.register_batch(list(F), list(M), cfg)
    with dreg.MultiContext([0]) as mc:
        mphis, mwarps, mres, rec = mc.register_batch(list(F), list(M), cfg)
    for i in range(5):
        assert np.array_equal(mphis[i], phis[i]) and np.array_equal(mwarps[i], warps[i])
        assert mres[i].velocity_count == res[i].velocity_count
        js = ctx.jacobian_stats(phis[i])
        r = rec[i]
        assert r.pair == i and r.device == 0 and r.status == 0
        assert r.velocity_count == res[i].velocity_count and r.solves == res[i].solves
        assert r.folding_voxels == js.nonpositive == res[i].folding_voxels
        assert r.min_det == pytest.approx(js.min_det, abs=0) and res[i].min_det == r.min_det
        lg = res[i].per_level[0]
        assert r.final_mean_sad == lg.mean_sad[lg.warps]
        assert r.admm_iterations == sum(lg.solver_iterations[w] for w in range(lg.warps))


@pytest.mark.gpu
def test_multi_rejects_bad_devices():
    with pytest.raises(RuntimeError):
        dreg.MultiContext([0, 0])
    with pytest.raises(RuntimeError):
        dreg.MultiContext([64])
