"""Frame sharding and the (only) collectives of the multi-GPU path.

Frames are independent (datagen batches of IR pairs, BASELINE.json north_star),
so rank r of N processes a contiguous frame range and nothing crosses GPUs on
the data path.  After the timed region: all_reduce(MAX) of the elapsed time and
all_gather of the per-frame statistics (asd_frame_stats: checksum, valid count,
depth sum) -- NCCL over NVLink on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations


def shard_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Frames [floor(r*B/N), floor((r+1)*B/N)) for rank r of N."""
    if world < 1 or not 0 <= rank < world or n_frames < 0:
        raise ValueError("bad shard arguments")
    return (rank * n_frames) // world, ((rank + 1) * n_frames) // world


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timer) across the default process group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_frame_stats(stats):
    """all_gather of equally sized per-rank [n, 4] int32 stats tensors -> [world*n, 4]."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return stats
    out = torch.empty((dist.get_world_size() * stats.shape[0],) + tuple(stats.shape[1:]),
                      dtype=stats.dtype, device=stats.device)
    dist.all_gather_into_tensor(out, stats.contiguous())
    return out
