"""World-size-2 gloo test of the multi-GPU plumbing (paper_2109_12688_b200/shard.py):
disjoint pair sharding, all-gather of per-pair records in rank order, MAX timing.
Runs on CPU; the GPU box uses the same code over NCCL."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_12688_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seeds = shard.pair_seeds(rank, world, per_rank)
        rec = torch.tensor([[0, 5 + rank, 6, 0, 0.01 * s, 0.3 + rank] for s in seeds], dtype=torch.float64)
        allrec = shard.gather_records(rec)
        t = shard.max_over_ranks(1.0 + rank)
        q.put((rank, seeds, allrec.numpy().tolist(), t))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather():
    world, per_rank = 2, 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seeds0, seeds1 = res[0][1], res[1][1]
    assert not set(seeds0) & set(seeds1)
    assert seeds0 == [1000, 1001, 1002] and seeds1 == [1003, 1004, 1005]
    for rank, _, allrec, t in res:
        assert len(allrec) == world * per_rank
        assert [r[1] for r in allrec] == [5] * 3 + [6] * 3  # rank-major order
        assert t == 2.0  # max over ranks
    summ = shard.summarize(torch.tensor(res[0][2], dtype=torch.float64))
    assert summ["count"] == 6 and summ["status_ok"] == 6 and summ["min_det"] == 0.3


def test_pair_seeds_cover_config3_pool():
    allseeds = [s for r in range(8) for s in shard.pair_seeds(r, 8, 32)]
    assert sorted(allseeds) == list(range(1000, 1256))
    with pytest.raises(ValueError):
        shard.pair_seeds(3, 2, 4)
