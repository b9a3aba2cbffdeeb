"""Multi-GPU plumbing for batched registration.

Independent image pairs are sharded by rank; no field data ever crosses devices.
The only collectives are an all-gather of fixed-size per-pair records (status,
velocity_count, solves, folding count, final mean SAD, min det J) and a MAX
all-reduce of the timed region -- torch.distributed over NCCL on the GPU box,
gloo in the CPU tests.
"""
from __future__ import annotations

RECORD_FIELDS = ("status", "velocity_count", "solves", "folding_voxels", "final_mean_sad", "min_det")


def pair_seeds(rank: int, world: int, per_rank: int, base: int = 1000) -> list[int]:
    """Seeds of `per_rank` pairs for `rank`: contiguous block base + rank * per_rank + i.
    Blocks of different ranks never overlap (8 ranks x 32 pairs = config 3's pool
    1000..1255)."""
    if per_rank < 0 or rank < 0 or rank >= max(world, 1):
        raise ValueError("bad rank/world/per_rank")
    start = base + rank * per_rank
    return list(range(start, start + per_rank))


def split_pairs(rank: int, world: int, total: int, base: int = 1000) -> list[int]:
    """Strong scaling: `total` pairs (seeds base..base+total-1) dealt to `world` ranks
    in contiguous blocks whose sizes differ by at most one (config 3: 256 / N)."""
    if total < 0 or world < 1 or rank < 0 or rank >= world:
        raise ValueError("bad rank/world/total")
    lo = (rank * total) // world
    hi = ((rank + 1) * total) // world
    return list(range(base + lo, base + hi))


def rank_seeds(rank: int, world: int, pairs: int, weak: bool, base: int = 1000) -> list[int]:
    """bench.py's dealing: strong (default) splits `pairs` over the ranks; weak gives
    every rank `pairs` distinct pairs of its own."""
    return pair_seeds(rank, world, pairs, base) if weak else split_pairs(rank, world, pairs, base)


def gather_records(records):
    """All-gather a [pairs, len(RECORD_FIELDS)] float64 tensor across ranks (rank-major).
    Ranks may hold different pair counts (strong scaling with N not dividing the
    total): counts are exchanged first and the records padded to the largest."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return records
    world = dist.get_world_size()
    n = torch.tensor([records.shape[0]], dtype=torch.int64, device=records.device)
    counts = torch.empty(world, dtype=torch.int64, device=records.device)
    dist.all_gather_into_tensor(counts, n)
    counts = [int(c) for c in counts.cpu()]
    cap = max(counts)
    padded = torch.zeros((cap, records.shape[1]), dtype=records.dtype, device=records.device)
    padded[: records.shape[0]] = records
    out = torch.empty((world * cap, records.shape[1]), dtype=records.dtype, device=records.device)
    dist.all_gather_into_tensor(out, padded.contiguous())
    return torch.cat([out[r * cap: r * cap + counts[r]] for r in range(world)])


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a scalar (the driver's max-over-ranks timing rule)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def summarize(records) -> dict:
    """Per-run summary of gathered per-pair records."""
    r = records
    return {
        "count": int(r.shape[0]),
        "status_ok": int((r[:, 0] == 0).sum()),
        "mean_velocity_count": float(r[:, 1].mean()),
        "mean_solves": float(r[:, 2].mean()),
        "folding_voxels_total": int(r[:, 3].sum()),
        "mean_final_sad": float(r[:, 4].mean()),
        "min_det": float(r[:, 5].min()),
    }
