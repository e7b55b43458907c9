"""Multi-GPU sharding of the flood filtration (one process per GPU).

The cloud and its spatial grid are replicated on every rank; the simplices
of each dimension are dealt round-robin (simplex j -> rank j % world), which
balances the very uneven per-simplex costs statistically without a cost
model.  Each rank values its shard with fph_flood_interior, the shards are
all-gathered (NCCL over NVLink), and every rank runs the facet completion.
Batches of independent clouds are distributed whole (cloud b -> rank
b % world, batch.flood_cloud_batch): no collective inside a cloud.
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

    if world == 1 and (dist is None or not dist.is_initialized()):
        return mine[:n_total]
    per = (n_total + world - 1) // world
    buf = torch.full((per,), float("nan"), dtype=mine.dtype, device=mine.device)
    buf[: mine.shape[0]] = mine
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.stack(parts, dim=1).reshape(-1)[:n_total]


def shard_interior(pts, lms, by_dim, top: int, m: int, subset: bool, rank: int, world: int,
                   stream=None):
    """This rank's interior squared values {k: tensor} (fph_flood_shard).

    pts, lms: float64 CUDA tensors (n x d, n_L x d); by_dim[k]: int32 CUDA
    tensors (n_k x (k+1)).  Row i of the result for dim k is simplex
    rank + i * world.
    """
    import torch

    from . import _native

    lib = _native.require_gpu()
    dev = pts.device
    counts = torch.tensor([by_dim[k].shape[0] for k in range(top + 1)], dtype=torch.int64)
    outs = [None] + [torch.empty(max(len(shard_rows(int(counts[k]), world, rank)), 1),
                                 dtype=torch.float64, device=dev) for k in range(1, top + 1)]
    simp = [None] + [by_dim[k] for k in range(1, top + 1)]
    with torch.cuda.device(dev):  # the library allocates on the current device
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        _native.check(lib.fph_flood_shard(
            pts.data_ptr(), pts.shape[0], pts.shape[1], lms.data_ptr(), lms.shape[0], top,
            counts.data_ptr(), _native.ptr_array(simp, None), rank, world, m, 1 if subset else 0,
            _native.ptr_array(outs, None), _native.FPH_MEM_DEVICE, s))
    return {k: outs[k][: len(shard_rows(int(counts[k]), world, rank))] for k in range(1, top + 1)}


def complete(interior: dict, facets: dict, n0: int, top: int, subset: bool, stream=None):
    """Facet completion on the device: {k: squared values} from the gathered
    interior terms (vertices 0 in subset mode)."""
    import torch

    from . import _native

    lib = _native.require_gpu()
    dev = interior[1].device
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    if not subset:
        raise ValueError("sharded runs need landmarks that are cloud points")
    out = {0: torch.zeros(n0, dtype=torch.float64, device=dev)}
    with torch.cuda.device(dev):
        for k in range(1, top + 1):
            out[k] = torch.empty_like(interior[k])
            _native.check(lib.fph_flood_complete(
                interior[k].data_ptr(), facets[k].data_ptr(), interior[k].shape[0], k,
                out[k - 1].data_ptr(), out[k].data_ptr(), s))
    return out


def flood_sq_values_sharded(pts, lms, by_dim, facets, top: int, m: int, dist, subset=True,
                            interior_fn=None, complete_fn=None):
    """Multi-GPU flood values: this rank's share (fph_flood_shard), all-gather
    of the interior terms (NCCL), facet completion on every rank.

    interior_fn(rank, world) -> {k: 1-D tensor} and complete_fn(interior,
    facets, n0, top, subset) -> {k: tensor} default to the device calls; the
    CPU multi-process tests substitute host implementations."""
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    if interior_fn is None:
        def interior_fn(r, w):
            return shard_interior(pts, lms, by_dim, top, m, subset, r, w)
    mine = interior_fn(rank, world)
    interior = {k: gather_interleaved(mine[k], by_dim[k].shape[0], world, dist)
                for k in range(1, top + 1)}
    return (complete_fn or complete)(interior, facets, by_dim[0].shape[0], top, subset)
