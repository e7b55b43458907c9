"""Batches of independent clouds (BASELINE configs[3]: 512 ModelNet-shaped
100k-point clouds, 1k landmarks each, over 8 GPUs).

The reference values one cloud per build_flood_filtration call
(floodph/filtration.py:348) and parallelises inside it over batches of top
cells on a thread pool (filtration.py:256-267).  Here the unit of parallelism
across GPUs is the cloud: cloud b goes to rank b % world, whole (no
collective inside a cloud).  Per rank:

  1. farthest point sampling of all its clouds in ONE launch
     (fph_farthest_point_sampling_batched: CTA groups run different clouds);
  2. Delaunay of each landmark set on a host thread pool, overlapped with
  3. the flood values of each finished complex on the device
     (fph_flood_filtration, device memory, the cloud already resident).

Results are gathered to every rank in cloud order (small: one float64 per
simplex) when a process group is given.
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .delaunay import Triangulation, delaunay
from .parallel import shard_rows


class DeviceComplex:
    """Device buffers of one landmark complex for the C-ABI flood call:
    landmarks (n_L x d float64), simplices and facet links per dimension
    (int32), and output buffers; max_dim limits it to a skeleton."""

    def __init__(self, tri: Triangulation, device, max_dim: int | None = None):
        import torch

        self.top = tri.dim if max_dim is None else min(max_dim, tri.dim)
        self.dev = torch.device(device)
        self.lm = torch.from_numpy(np.ascontiguousarray(tri.points, dtype=np.float64)).to(self.dev)
        self.counts_full = [int(tri.simplices_by_dim[k].shape[0]) for k in range(self.top + 1)]
        self.counts = torch.tensor(self.counts_full, dtype=torch.int64)
        self.simp = {k: torch.from_numpy(np.ascontiguousarray(tri.simplices_by_dim[k],
                                                              dtype=np.int32)).to(self.dev)
                     for k in range(1, self.top + 1)}
        self.facets = {k: torch.from_numpy(np.ascontiguousarray(tri.facet_links[k],
                                                                dtype=np.int32)).to(self.dev)
                       for k in range(1, self.top + 1)}
        self.out = [torch.empty(max(c, 1), dtype=torch.float64, device=self.dev)
                    for c in self.counts_full]

    @property
    def n_simplices(self) -> int:
        return sum(self.counts_full)


def flood_sq_device(points, dc: DeviceComplex, m: int, subset: bool = True, stream=None):
    """Squared flood values of dc's complex over the device cloud `points`
    (n x d float64 CUDA tensor) into dc.out, ordered on `stream` (default:
    the current torch stream); returns dc.out trimmed per dimension."""
    import torch

    lib = _native.require_gpu()
    simp = [None] + [dc.simp[k] for k in range(1, dc.top + 1)]
    fac = [None] + [dc.facets[k] for k in range(1, dc.top + 1)]
    with torch.cuda.device(dc.dev):
        s = stream if stream is not None else torch.cuda.current_stream(dc.dev).cuda_stream
        _native.check(lib.fph_flood_filtration(
            points.data_ptr(), points.shape[0], points.shape[1], dc.lm.data_ptr(), dc.lm.shape[0],
            dc.top, dc.counts.data_ptr(), _native.ptr_array(simp, None),
            _native.ptr_array(fac, None), int(m), 1 if subset else 0,
            _native.ptr_array(dc.out, None), _native.FPH_MEM_DEVICE, s))
    return [dc.out[k][: dc.counts_full[k]] for k in range(dc.top + 1)]


_LANES: dict = {}


def _lane_streams(dev, lanes: int = 2):
    import torch

    key = (dev.index, lanes)
    if key not in _LANES:
        _LANES[key] = [torch.cuda.Stream(device=dev) for _ in range(lanes)]
    return _LANES[key]


def flood_sq_device_many(items, m: int, subset: bool = True, stream=None, lanes: int = 2):
    """Squared flood values of several (points, DeviceComplex) items, the
    calls dealt round-robin to `lanes` streams forked from `stream` (default:
    the current torch stream) and joined back into it: the next cloud's grid
    build and set-up run under the current cloud's search tail (a few heavy
    simplices on a few warps); the search kernels themselves take the
    device's grid slot in turn (FPH_GRID_SLOTS=2 lets them overlap too, see
    fph_api.cu GridSlot).  modelnet_batch: 163 -> 143 ms per 64 clouds.
    Returns each item's dc.out trimmed per dimension, in order."""
    import torch

    dev = items[0][1].dev
    with torch.cuda.device(dev):
        base = (torch.cuda.ExternalStream(stream, device=dev) if stream is not None
                else torch.cuda.current_stream(dev))
        side = _lane_streams(dev, lanes)
        for s in side:
            s.wait_stream(base)
        out = [flood_sq_device(X, dc, m, subset, side[i % lanes].cuda_stream)
               for i, (X, dc) in enumerate(items)]
        for s in side:
            base.wait_stream(s)
    return out


@dataclass
class CloudResult:
    """One cloud of a batch: landmark indices, complex, squared flood values."""

    cloud: int
    landmark_indices: np.ndarray
    triangulation: Triangulation
    sq_values: dict


@dataclass
class BatchReport:
    results: list
    timings: dict = field(default_factory=dict)


def flood_cloud_batch(clouds, n_landmarks: int, m: int = 20, max_dim: int | None = None,
                      start: int = 0, dist=None, device=None, workers: int | None = None,
                      gather: bool = True) -> BatchReport:
    """Flood values of every cloud of a (B, n, d) batch, clouds dealt
    round-robin to the ranks of `dist` (None: one process).

    Each rank runs one batched FPS launch over its clouds, triangulates the
    landmark sets on `workers` host threads and values each complex on its
    GPU as soon as it is triangulated.  With gather=True every rank returns
    all B results in cloud order, else only its own."""
    import torch

    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    X = clouds if isinstance(clouds, torch.Tensor) else torch.from_numpy(np.asarray(clouds, dtype=np.float64))
    if X.dim() != 3:
        raise ValueError("expected a (batch, n, dim) stack of clouds")
    mine = shard_rows(X.shape[0], world, rank)
    timings = {"fps_s": 0.0, "delaunay_s": 0.0, "flood_s": 0.0}
    results = []
    if mine.size:
        from .geometry import farthest_point_sampling_batched

        Xd = X[torch.from_numpy(mine)].to(dev).contiguous()
        t0 = time.perf_counter()
        idx = farthest_point_sampling_batched(Xd, n_landmarks, start).cpu().numpy()
        timings["fps_s"] = time.perf_counter() - t0
        Xh = X[torch.from_numpy(mine)].cpu().numpy() if X.is_cuda else X.numpy()[mine]

        def triangulate(i):
            t = time.perf_counter()
            tri = delaunay(Xh[i][idx[i]])
            return tri, time.perf_counter() - t

        pending = []
        with ThreadPoolExecutor(max_workers=workers or 4) as pool:
            futures = [pool.submit(triangulate, i) for i in range(len(mine))]
            for i, fut in enumerate(futures):
                tri, dt = fut.result()
                timings["delaunay_s"] += dt
                t0 = time.perf_counter()
                dc = DeviceComplex(tri, dev, max_dim)
                # queued on alternating streams: two clouds in flight
                lane = _lane_streams(dev)[i % 2]
                lane.wait_stream(torch.cuda.current_stream(dev))
                sq = flood_sq_device(Xd[i], dc, m, True, lane.cuda_stream)
                pending.append((i, tri, dc, sq, lane))
                timings["flood_s"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        for i, tri, dc, sq, s in pending:
            s.synchronize()
            vals = {k: v.cpu().numpy() for k, v in enumerate(sq)}
            results.append(CloudResult(int(mine[i]), idx[i], tri, vals))
        timings["flood_s"] += time.perf_counter() - t0
    if gather and world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, results)
        results = sorted((r for p in parts for r in p), key=lambda r: r.cloud)
    return BatchReport(results=results, timings=timings)
