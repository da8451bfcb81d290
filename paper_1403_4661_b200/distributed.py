"""Multi-GPU data parallelism over maps: one process per GPU (torch.distributed).

Maps are independent, so a batch is split into contiguous shards, each rank
transforms its shard on its own GPU, and (optionally) the shards are gathered
back -- no collective on the transform's data path itself (the
order-sharded single-map path with an NCCL exchange between sweep blocks is
future work).  Timings are reduced as the max over ranks.
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) shard of `total` items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a scalar over all ranks (timing rule: device time, max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sharded_apply(batch: np.ndarray, compute: Callable[[np.ndarray], np.ndarray], group=None,
                  gather: bool = True) -> np.ndarray:
    """Split `batch` (B, L^2) over ranks, run `compute` on the local shard, all-gather.

    `compute` is the per-rank transform (e.g. ``lambda x: inverse_sht_batch(x, grid,
    device=local_rank)``); every rank passes the same full batch.  With
    ``gather=False`` the local shard's result is returned.
    """
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return compute(batch)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_bounds(batch.shape[0], rank, world)
    local = np.ascontiguousarray(compute(batch[lo:hi])) if hi > lo else np.empty((0,) + batch.shape[1:],
                                                                                  batch.dtype)
    if not gather:
        return local
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    width = max(b - a for a, b in (shard_bounds(batch.shape[0], r, world) for r in range(world)))
    buf = torch.zeros((width,) + batch.shape[1:], dtype=torch.complex128, device=dev)
    if hi > lo:
        buf[: hi - lo] = torch.from_numpy(local).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = []
    for r in range(world):
        a, b = shard_bounds(batch.shape[0], r, world)
        out.append(parts[r][: b - a].cpu().numpy())
    return np.concatenate(out, axis=0)
