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


# ---------------------------------------------------------------- spatial shards
def simplex_centers(landmarks: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Ritter centers (midpoint of the first longest edge) of the simplices
    `rows` (n x (k+1) landmark ids): the same rule as the device code, used
    only to place simplices in space for partitioning."""
    V = np.asarray(landmarks, dtype=np.float64)[np.asarray(rows)]
    k1 = V.shape[1]
    if k1 == 1:
        return V[:, 0, :]
    best = np.full(V.shape[0], -1.0)
    c = np.zeros((V.shape[0], V.shape[2]))
    for i in range(k1):
        for j in range(i + 1, k1):
            d = ((V[:, i] - V[:, j]) ** 2).sum(axis=1)
            upd = d > best
            best[upd] = d[upd]
            c[upd] = 0.5 * (V[upd, i] + V[upd, j])
    return c


def morton_order(centers: np.ndarray) -> np.ndarray:
    """Permutation sorting points along a 30-bit Morton (Z-order) curve of
    their bounding box (stable: ties keep row order)."""
    c = np.asarray(centers, dtype=np.float64)
    if c.shape[0] == 0:
        return np.zeros(0, dtype=np.int64)
    lo = c.min(axis=0)
    ext = max(float((c.max(axis=0) - lo).max()), 1e-300)
    q = np.clip(((c - lo) / ext * 1023.0).astype(np.int64), 0, 1023)
    code = np.zeros(c.shape[0], dtype=np.int64)
    for bit in range(10):
        for a in range(c.shape[1]):
            code |= ((q[:, a] >> bit) & 1) << (bit * c.shape[1] + a)
    return np.argsort(code, kind="stable")


def spatial_partition(centers: np.ndarray, costs, world: int) -> list:
    """Cut the Morton order of the simplex centers into `world` contiguous
    pieces of (nearly) equal total cost: each rank's simplices are spatially
    compact, so its share of the cloud stays in L2.  Deterministic (every
    rank computes the same partition).  Returns per-rank row arrays."""
    order = morton_order(centers)
    w = np.ones(order.shape[0]) if costs is None else np.asarray(costs, dtype=np.float64)[order]
    cum = np.cumsum(w)
    total = cum[-1] if cum.size else 0.0
    cuts = np.searchsorted(cum, total * np.arange(1, world) / world, side="right")
    return [np.sort(part) for part in np.split(order, cuts)]


def subset_interior(pts, lms, by_dim, top: int, m: int, subset: bool, rows: dict, stream=None):
    """Interior squared values {k: tensor} of the listed rows of each
    dimension (fph_flood_subset, one grid build); rows[k]: int64 CUDA tensor."""
    import torch

    from . import _native

    lib = _native.require_gpu()
    dev = pts.device
    counts = torch.tensor([by_dim[k].shape[0] for k in range(top + 1)], dtype=torch.int64)
    nrows = torch.tensor([0] + [int(rows[k].shape[0]) for k in range(1, top + 1)], dtype=torch.int64)
    outs = [None] + [torch.empty(max(int(nrows[k]), 1), dtype=torch.float64, device=dev)
                     for k in range(1, top + 1)]
    simp = [None] + [by_dim[k] for k in range(1, top + 1)]
    rws = [None] + [rows[k] for k in range(1, top + 1)]
    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        _native.check(lib.fph_flood_subset(
            pts.data_ptr(), pts.shape[0], pts.shape[1], lms.data_ptr(), lms.shape[0], top,
            counts.data_ptr(), _native.ptr_array(simp, None), _native.ptr_array(rws, None),
            nrows.data_ptr(), m, 1 if subset else 0, _native.ptr_array(outs, None),
            _native.FPH_MEM_DEVICE, s))
    return {k: outs[k][: int(nrows[k])] for k in range(1, top + 1)}


def gather_partitioned(mine, parts, n_total: int, world: int, dist):
    """All-gather every rank's values for its rows parts[r] (a list of
    int64 device tensors, the same on every rank) into row order."""
    import torch

    full = torch.empty(n_total, dtype=mine.dtype, device=mine.device)
    if world == 1 and (dist is None or not dist.is_initialized()):
        full[parts[0]] = mine
        return full
    per = max(int(p.shape[0]) for p in parts)
    buf = torch.full((per,), float("nan"), dtype=mine.dtype, device=mine.device)
    buf[: mine.shape[0]] = mine
    got = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(got, buf)
    for r in range(world):
        full[parts[r]] = got[r][: parts[r].shape[0]]
    return full


def flood_sq_values_spatial(pts, lms, by_dim, facets, top: int, m: int, dist, parts: dict,
                            subset=True):
    """Multi-GPU flood values over spatially compact shards: parts[k][r] are
    the rows of dimension k valued by rank r (spatial_partition), the shares
    all-gathered (NCCL) and completed on every rank."""
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    mine = subset_interior(pts, lms, by_dim, top, m, subset, {k: parts[k][rank] for k in range(1, top + 1)})
    interior = {k: gather_partitioned(mine[k], parts[k], by_dim[k].shape[0], world, dist)
                for k in range(1, top + 1)}
    return complete(interior, facets, by_dim[0].shape[0], top, subset)
