"""Multi-GPU sharding of the flood filtration (one process per GPU).

The cloud and its spatial grid are replicated on every rank; the simplices
of each dimension are dealt round-robin (simplex j -> rank j % world), which
balances the very uneven per-simplex costs statistically without a cost
model.  Each rank values its shard with fph_flood_interior, the shards are
all-gathered (NCCL over NVLink), and every rank runs the facet completion.
Batches of independent clouds (farthest point sampling) are distributed
whole: cloud b -> rank b % world.
"""

from __future__ import annotations

import numpy as np


def shard_rows(n: int, world: int, rank: int) -> np.ndarray:
    """Rows of an n-row array owned by `rank` (interleaved)."""
    if not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    return np.arange(rank, n, world)


def gather_interleaved(mine, n_total: int, world: int, dist):
    """All-gather interleaved shards back into original row order.

    `mine` holds rows rank, rank + world, ... (a 1-D tensor on the process
    group's device).  Shards are padded to equal length for all_gather.
    """
    import torch

    if world == 1:
        return mine[:n_total]
    per = (n_total + world - 1) // world
    buf = torch.full((per,), float("nan"), dtype=mine.dtype, device=mine.device)
    buf[: mine.shape[0]] = mine
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.stack(parts, dim=1).reshape(-1)[:n_total]


def shard_clouds(batch: int, world: int, rank: int) -> np.ndarray:
    """Cloud ids of a batch owned by `rank` (whole clouds, round-robin)."""
    return shard_rows(batch, world, rank)
