"""Multi-GPU plumbing for batched registration.

Independent image pairs are sharded by rank; no field data ever crosses devices.
The only collectives are an all-gather of fixed-size per-pair records (status,
velocity_count, solves, folding count, final mean SAD, min det J) and a MAX
all-reduce of the timed region -- torch.distributed over NCCL on the GPU box,
gloo in the CPU tests.
"""
from __future__ import annotations

RECORD_FIELDS = ("status", "velocity_count", "solves", "folding_voxels", "final_mean_sad", "min_det")


def pair_seeds(rank: int, world: int, per_rank: int, base: int = 1000, pool: int = 256) -> list[int]:
    """Seeds of the pairs a rank registers: config 3's pool 1000..1255, dealt in
    contiguous blocks of `per_rank` (8 ranks x 32 pairs = the whole pool)."""
    if per_rank < 0 or rank < 0 or rank >= max(world, 1):
        raise ValueError("bad rank/world/per_rank")
    start = rank * per_rank
    return [base + (start + i) % pool for i in range(per_rank)]


def gather_records(records):
    """All-gather a [pairs, len(RECORD_FIELDS)] float64 tensor across ranks (rank-major)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return records
    world = dist.get_world_size()
    out = torch.empty((world * records.shape[0], records.shape[1]), dtype=records.dtype, device=records.device)
    dist.all_gather_into_tensor(out, records.contiguous())
    return out


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
