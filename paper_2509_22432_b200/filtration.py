"""Flood filtration of the landmark Delaunay complex, computed on the GPU.

Drop-in for reference floodph/filtration.py:348 build_flood_filtration: the
same inputs (cloud, landmark count or landmark array, FloodConfig), the same
FilteredComplex (simplices grouped by dimension, lexicographic, with values,
the (value, dim, vertices) total order and stage timings in meta).  The
per-simplex values come from one C-ABI call, fph_flood_filtration
(include/floodph_b200.h), which runs the grid build, the flooding kernel for
every dimension and the facet completion on the device; there is no CPU
fallback.  Values are bit-identical to the reference's float64 values.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from itertools import combinations

import numpy as np

from . import _native
from .delaunay import Triangulation, delaunay
from .errors import IntegrityError
from .geometry import (PointCloud, as_points, farthest_point_sampling, grid_covering_bound,
                       ritter_enclosing_ball)
from .spatial import AxisSortedCloud, slab_indices

STAGE_LANDMARKS = "Landmark select."
STAGE_DELAUNAY = "Delaunay triang."
STAGE_MASKING = "Masking"
STAGE_FILTRATION = "Filtration"

SAMPLERS = ("grid", "uniform-random")
# the reference's two CPU strategies both map to the one exact device path
BACKENDS = ("masked-batch", "kdtree", "cuda")


@dataclass(frozen=True)
class FloodConfig:
    """Reference knobs (floodph/filtration.py:51) plus `max_dim`.

    grid_resolution m puts C(m+k, k) sample points on a k-simplex.
    batch_size and threads are accepted for compatibility; the device path's
    scheduling does not depend on them (results never did).  max_dim limits
    the complex to its max_dim-skeleton (None: the full Delaunay complex, as
    the reference); values of the kept simplices are unchanged.
    """

    grid_resolution: int = 20
    batch_size: int = 256
    sampler: str = "grid"
    sampler_count: int = 100
    sampler_seed: int = 0
    backend: str = "masked-batch"
    fps_start: int = 0
    delaunay_seed: int = 0
    threads: int | None = None
    max_dim: int | None = None

    def validate(self) -> None:
        if self.grid_resolution < 1:
            raise ValueError("grid_resolution must be >= 1")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.sampler not in SAMPLERS:
            raise ValueError(f"sampler must be one of {SAMPLERS}")
        if self.sampler_count < 1:
            raise ValueError("sampler_count must be >= 1")
        if self.backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}")
        if self.threads is not None and self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.max_dim is not None and not 0 <= self.max_dim <= 3:
            raise ValueError("max_dim must be in [0, 3]")


@dataclass(frozen=True)
class CandidateMask:
    """Per simplex of a batch: the ascending cloud indices inside its masking
    ball (|x - c|^2 <= 2 r^2, (c, r) its Ritter ball).  Reference
    floodph/filtration.py:88."""

    simplices: np.ndarray
    candidates: list


@dataclass(frozen=True)
class FilteredComplex:
    """simplices: (vertex tuple, dim, value) grouped by dim, lexicographic;
    order[i]: rank of simplices[i] under (value, dim, vertex tuple)."""

    simplices: list
    order: np.ndarray
    meta: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return len(self.simplices)

    def in_order(self) -> list:
        ranked = [None] * len(self.simplices)
        for i, r in enumerate(self.order):
            ranked[r] = self.simplices[i]
        return ranked

    def value_map(self) -> dict:
        return {verts: value for verts, _, value in self.simplices}


def compute_mask(triangulation: Triangulation, X, sorted_cloud: AxisSortedCloud,
                 batch) -> CandidateMask:
    """Candidate cloud indices of each simplex of `batch` (rows of landmark ids
    into triangulation.points), from the device grid (fph_candidate_mask).

    Same result as reference floodph/filtration.py:130: every cloud point of
    the closed ball |x - c|^2 <= 2 r r, ascending.  An empty ball (possible
    only for landmarks away from the cloud) falls back, as in the reference,
    to the batch's axis slab (bounds: extreme center -+ sqrt(2) r (1 + 1e-12)
    along sorted_cloud.axis), then to the whole cloud.
    """
    pts = np.ascontiguousarray(as_points(X), dtype=np.float64)
    cells = np.asarray(batch, dtype=np.int64)
    if cells.ndim == 1:
        cells = cells.reshape(1, -1)
    if cells.shape[0] == 0:
        return CandidateMask(cells, [])
    if cells.shape[1] < 2:
        raise ValueError("enclosing ball needs at least 2 vertices")
    if cells.shape[1] > 4:
        raise ValueError("simplices of dimension above 3 are not supported")
    lib = _native.require_gpu()
    lms = np.ascontiguousarray(triangulation.points, dtype=np.float64)
    c32 = np.ascontiguousarray(cells, dtype=np.int32)
    k = cells.shape[1] - 1
    offs = np.zeros(cells.shape[0] + 1, dtype=np.int64)
    args = (_native.ptr(pts), pts.shape[0], pts.shape[1], _native.ptr(lms), lms.shape[0],
            _native.ptr(c32), cells.shape[0], k, _native.ptr(offs))
    _native.check(lib.fph_candidate_mask(*args, None, 0))
    idx = np.empty(max(int(offs[-1]), 1), dtype=np.int32)
    _native.check(lib.fph_candidate_mask(*args, _native.ptr(idx), idx.shape[0]))
    idx = idx.astype(np.int64)
    candidates = [idx[offs[i]:offs[i + 1]] for i in range(cells.shape[0])]
    if any(c.size == 0 for c in candidates):
        balls = [ritter_enclosing_ball(lms[c]) for c in cells]
        axis = sorted_cloud.axis
        spans = [math.sqrt(2.0) * b.radius * (1.0 + 1e-12) for b in balls]
        lo = min(b.center[axis] - sp for b, sp in zip(balls, spans))
        hi = max(b.center[axis] + sp for b, sp in zip(balls, spans))
        slab = np.sort(slab_indices(sorted_cloud, lo, hi))
        fallback = slab if slab.size else np.arange(pts.shape[0], dtype=np.int64)
        candidates = [c if c.size else fallback for c in candidates]
    return CandidateMask(cells, candidates)


def _max_min_sq(grid_points: np.ndarray, cloud: np.ndarray) -> float:
    """max over grid rows of the min squared distance to the cloud (GPU:
    the rows as explicit samples of one 0-simplex at their centroid, the
    whole cloud searched)."""
    lib = _native.require_gpu()
    g = np.ascontiguousarray(grid_points, dtype=np.float64)
    c = np.ascontiguousarray(cloud, dtype=np.float64)
    center = np.ascontiguousarray(g.mean(axis=0, keepdims=True))
    s4 = np.array([[0, -1, -1, -1]], dtype=np.int32)
    out = np.empty(1)
    _native.check(lib.fph_flood_samples(
        _native.ptr(c), c.shape[0], c.shape[1], _native.ptr(center), 1, _native.ptr(s4), 1, 0,
        _native.ptr(g), g.shape[0], 0, _native.ptr(out), _native.FPH_MEM_HOST, None))
    return float(out[0])


def simplex_filtration(simplex, grid_points: np.ndarray, candidates, X) -> float:
    """max over the grid points of the min distance to X[candidates] (GPU).
    Reference floodph/filtration.py:165; candidates must be non-empty."""
    cand = np.asarray(candidates, dtype=np.int64)
    if cand.size == 0:
        raise IntegrityError(f"empty candidate set for simplex {tuple(simplex)}")
    grid = as_points(grid_points)
    if grid.shape[0] == 0:
        raise ValueError("empty grid")
    return math.sqrt(_max_min_sq(grid, as_points(X)[cand]))


def _simplex_closure(k: int):
    """All faces of the standard k-simplex {0..k}, by dimension, with their
    facet links (the Triangulation layout)."""
    by_dim = {j: np.array(list(combinations(range(k + 1), j + 1)), dtype=np.int64)
              for j in range(k + 1)}
    links = {}
    for j in range(1, k + 1):
        lower = {tuple(r): i for i, r in enumerate(by_dim[j - 1].tolist())}
        links[j] = np.array([[lower[tuple(r[:t] + r[t + 1:])] for t in range(j + 1)]
                             for r in by_dim[j].tolist()], dtype=np.int64)
    return by_dim, links


def flood_value_exact_gap(simplex, m: int, X) -> tuple:
    """(value of the resolution-m grid of the simplex, that + the grid's
    covering bound): brackets the continuous flood value.  Reference
    floodph/filtration.py:178.  The grid value is the flood filtration of the
    simplex's own closure on the GPU (every row of the full grid: interior
    rows of each face, then facet completion), over the whole cloud."""
    verts = np.ascontiguousarray(as_points(simplex), dtype=np.float64)
    pts = np.ascontiguousarray(as_points(X), dtype=np.float64)
    if m < 1:
        raise ValueError("resolution must be at least 1")
    k = verts.shape[0] - 1
    if k < 0 or k > 3:
        raise ValueError("simplices of dimension 0..3 are supported")
    if verts.shape[1] != pts.shape[1]:
        raise ValueError("simplex and cloud dimensions differ")
    by_dim, links = _simplex_closure(k)
    tri = Triangulation(dim=k, points=verts, vertices=np.arange(k + 1), simplices_by_dim=by_dim,
                        facet_links=links, dedup_dropped=np.zeros(0, np.int64),
                        jitter_applied=False, warnings=())
    subset = _landmarks_in_cloud(verts, pts)
    sq = flood_sq_values(pts, tri, int(m), subset)
    f = math.sqrt(float(sq[k][0]))
    return f, f + grid_covering_bound(verts, m)


def _landmarks_in_cloud(landmarks: np.ndarray, pts: np.ndarray) -> bool:
    """Every landmark row equals some cloud row bit for bit."""
    if landmarks.shape[1] != pts.shape[1]:
        return False
    dt = np.dtype((np.void, pts.dtype.itemsize * pts.shape[1]))
    cloud = np.ascontiguousarray(pts).view(dt).ravel()
    lm = np.ascontiguousarray(landmarks).view(dt).ravel()
    return bool(np.isin(lm, cloud).all())


def flood_sq_values(pts: np.ndarray, tri: Triangulation, m: int, subset: bool,
                    max_dim: int | None = None) -> dict:
    """Squared flood values {k: (n_k,) float64} of the complex, via the C ABI."""
    top = tri.dim if max_dim is None else min(max_dim, tri.dim)
    lib = _native.require_gpu()
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    lms = np.ascontiguousarray(tri.points, dtype=np.float64)
    counts = np.array([tri.simplices_by_dim[k].shape[0] for k in range(top + 1)], dtype=np.int64)
    simp = [None] + [np.ascontiguousarray(tri.simplices_by_dim[k], dtype=np.int32)
                     for k in range(1, top + 1)]
    fac = [None] + [np.ascontiguousarray(tri.facet_links[k], dtype=np.int32)
                    for k in range(1, top + 1)]
    outs = [np.empty(max(int(c), 1)) for c in counts]
    _native.check(lib.fph_flood_filtration(
        _native.ptr(pts), pts.shape[0], pts.shape[1], _native.ptr(lms), lms.shape[0], top,
        _native.ptr(counts), _native.ptr_array(simp, None), _native.ptr_array(fac, None),
        int(m), 1 if subset else 0, _native.ptr_array(outs, None),
        _native.FPH_MEM_HOST, None))
    return {k: outs[k][: counts[k]] for k in range(top + 1)}


def _check_monotone(values: dict, tri: Triangulation) -> None:
    for k in range(1, max(values) + 1):
        facet_vals = values[k - 1][tri.facet_links[k]]
        bad = facet_vals > values[k][:, None]
        if bad.any():
            raise IntegrityError(f"filtration not monotone: {int(bad.sum())} face pair(s) in dim {k}")


def filtration_order(values: dict, by_dim: dict) -> np.ndarray:
    """Rank of each simplex (grouped-by-dim order) under (value, dim, vertices)."""
    vals = np.concatenate([values[k] for k in sorted(values)])
    dims = np.concatenate([np.full(values[k].shape[0], k) for k in sorted(values)])
    width = max(values) + 1
    verts = np.full((vals.shape[0], width), -1, dtype=np.int64)
    row = 0
    for k in sorted(values):
        rows = by_dim[k]
        verts[row:row + rows.shape[0], : k + 1] = rows
        row += rows.shape[0]
    # lexsort: last key is primary; shorter tuples only compare within a dim
    keys = [verts[:, c] for c in range(width - 1, -1, -1)] + [dims, vals]
    ranks = np.lexsort(keys)
    order = np.empty(vals.shape[0], dtype=np.int64)
    order[ranks] = np.arange(vals.shape[0])
    return order


def build_flood_filtration(X, L, config: FloodConfig | None = None) -> FilteredComplex:
    """Landmarks -> Delaunay -> flood value of every simplex (GPU).

    L: a landmark count (farthest point sampling from config.fps_start, on
    the GPU) or an explicit (k, d) landmark array.  Landmarks that are cloud
    points get the pruned search (Lemma 4.2) and vertex value 0; others are
    searched against the whole cloud and vertices get d(v, X), as the
    reference's kdtree route.
    """
    config = config or FloodConfig()
    config.validate()
    if config.sampler != "grid":
        from .sampling import random_sampler_values  # uniform-random sampler
    cloud = X if isinstance(X, PointCloud) else PointCloud(np.asarray(X, dtype=np.float64))
    pts = cloud.points
    meta = {"config": config}
    timings = {STAGE_LANDMARKS: 0.0, STAGE_DELAUNAY: 0.0, STAGE_MASKING: 0.0,
               STAGE_FILTRATION: 0.0}

    t0 = time.perf_counter()
    if isinstance(L, (int, np.integer)):
        idx = farthest_point_sampling(pts, int(L), start=config.fps_start)
        landmarks = pts[idx]
        subset = True
        meta["landmark_indices"] = idx
    else:
        landmarks = as_points(L)
        subset = _landmarks_in_cloud(landmarks, pts)
    meta["landmark_mode"] = "subset" if subset else "external"
    timings[STAGE_LANDMARKS] = time.perf_counter() - t0

    t0 = time.perf_counter()
    tri = delaunay(landmarks, seed=config.delaunay_seed)
    timings[STAGE_DELAUNAY] = time.perf_counter() - t0
    meta["triangulation"] = tri
    meta["warnings"] = list(tri.warnings)
    meta["backend"] = "cuda"
    if not subset:
        meta["warnings"].append(
            "landmarks are not a subset of the cloud; pruning is unsound, searching the whole cloud")

    top = tri.dim if config.max_dim is None else min(config.max_dim, tri.dim)
    t0 = time.perf_counter()
    if config.sampler == "grid":
        sq = flood_sq_values(pts, tri, config.grid_resolution, subset, top)
        for k, v in sq.items():
            if np.isnan(v).any():
                raise IntegrityError(f"unvalued simplices in dimension {k}")
        values = {k: np.sqrt(v) for k, v in sq.items()}
    else:
        values = random_sampler_values(pts, tri, config, subset, top)
    timings[STAGE_FILTRATION] = time.perf_counter() - t0
    _check_monotone(values, tri)
    meta["timings"] = timings

    simplices = []
    for k in range(top + 1):
        vals = values[k]
        for i, row in enumerate(tri.simplices_by_dim[k].tolist()):
            simplices.append((tuple(row), k, float(vals[i])))
    order = filtration_order(values, tri.simplices_by_dim)
    return FilteredComplex(simplices=simplices, order=order, meta=meta)
