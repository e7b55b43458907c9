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

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .delaunay import Triangulation, delaunay
from .errors import IntegrityError
from .geometry import PointCloud, as_points, farthest_point_sampling

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
        if self.grid_resolution > 255:
            raise ValueError("grid_resolution must be <= 255")
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
