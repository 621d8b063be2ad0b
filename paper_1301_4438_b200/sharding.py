"""Batch sharding across ranks (one process per GPU) — no data-path collective.

Independent matrices of a batch are split by rank; the only communication is the
timing / work reduction used for reporting (max of per-rank device time, sum of
per-rank work), and an optional gather of ranks/permutations for callers that want
the global result on one rank.  torch.distributed provides the process group
(NCCL on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of `total` items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_seed(base_seed: int, rank: int) -> int:
    """Seed of a rank's synthetic shard in weak scaling (each rank draws its own batch)."""
    return int(base_seed) + int(rank)


def reduce_timing(seconds: float, work: float, device=None):
    """(max seconds over ranks, sum of work over ranks); identity without a process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(seconds), float(work)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([seconds], dtype=torch.float64, device=dev)
    w = torch.tensor([work], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t.item()), float(w.item())


def gather_ranks(local_ranks: np.ndarray, total: int, device=None) -> np.ndarray:
    """All-gather the per-matrix ranks of every shard into the global order."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return np.asarray(local_ranks, dtype=np.int64)
    world = dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    sizes = [shard_range(total, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    buf = torch.full((width,), -1, dtype=torch.int64, device=dev)
    buf[: len(local_ranks)] = torch.as_tensor(np.asarray(local_ranks, dtype=np.int64), device=dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    parts = [out[r][: hi - lo].cpu().numpy() for r, (lo, hi) in enumerate(sizes)]
    return np.concatenate(parts)
