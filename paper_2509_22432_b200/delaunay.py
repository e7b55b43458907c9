"""Delaunay triangulation of the landmark set (host side, qhull).

The reference builds Del(L) with scipy's qhull (floodph/delaunay.py:105) and
so does this package: the triangulation is small (|L| <= ~10^4) and stays on
the host, timed as its own stage.  The policy around the qhull call is the
reference's, so both produce the same complex for the same landmarks:
duplicates dropped (first occurrence kept), affinely deficient input
rejected, and a seeded relative jitter (1e-12, 1e-11, 1e-10) retried when
qhull leaves points out or the unjittered cells are not in general position.
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import combinations

import numpy as np
from scipy.spatial import Delaunay as _Qhull
from scipy.spatial import QhullError, cKDTree

from .errors import DegeneracyError
from .geometry import as_points

JITTER_SCALE = 1e-12
GP_TOL = 1e-9


@dataclass(frozen=True)
class Triangulation:
    """simplices_by_dim[k]: (n_k, k+1) int rows, sorted, lexicographic;
    facet_links[k][i, j]: row in dim k-1 of simplex i without vertex j;
    points: deduplicated landmark coordinates; vertices: their original ids."""

    dim: int
    points: np.ndarray
    vertices: np.ndarray
    simplices_by_dim: dict
    facet_links: dict
    dedup_dropped: np.ndarray
    jitter_applied: bool
    warnings: tuple

    @property
    def top_cells(self) -> np.ndarray:
        return self.simplices_by_dim[self.dim]

    def counts(self) -> dict:
        return {k: int(v.shape[0]) for k, v in self.simplices_by_dim.items()}


def _first_occurrences(pts: np.ndarray):
    keys = [row.tobytes() for row in pts]
    first = {}
    keep, drop = [], []
    for i, key in enumerate(keys):
        if key in first:
            drop.append(i)
        else:
            first[key] = i
            keep.append(i)
    return np.asarray(keep, dtype=np.int64), np.asarray(drop, dtype=np.int64)


def circumcenters(points: np.ndarray, cells: np.ndarray):
    """Circumcenter and radius of each full-dimensional cell (inf if flat)."""
    dim = points.shape[1]
    centers = np.empty((cells.shape[0], dim))
    radii = np.empty(cells.shape[0])
    for i, cell in enumerate(cells):
        v = points[cell]
        e = v[1:] - v[0]
        rhs = 0.5 * np.einsum("ij,ij->i", e, e)
        try:
            y = np.linalg.solve(e @ e.T, rhs)
        except np.linalg.LinAlgError:
            centers[i] = np.nan
            radii[i] = np.inf
            continue
        c = v[0] + y @ e
        centers[i] = c
        radii[i] = float(np.linalg.norm(c - v[0]))
    return centers, radii


def _general_position_violated(pts: np.ndarray, cells: np.ndarray) -> bool:
    centers, radii = circumcenters(pts, cells)
    if not np.isfinite(radii).all():
        return True
    tree = cKDTree(pts)
    slack = GP_TOL * max(1.0, float(np.abs(pts).max()))
    need = pts.shape[1] + 1
    return any(len(tree.query_ball_point(c, r + slack)) > need for c, r in zip(centers, radii))


def _qhull_cells(work: np.ndarray):
    tri = _Qhull(work)
    if len(tri.coplanar):
        raise QhullError("qhull left coplanar points out of the triangulation")
    return tri.simplices


def _close_faces(cells: np.ndarray, dim: int):
    by_dim = {}
    for k in range(dim + 1):
        if k == dim:
            faces = cells
        else:
            faces = np.concatenate([cells[:, list(c)] for c in combinations(range(dim + 1), k + 1)])
        by_dim[k] = np.unique(faces, axis=0)
    links = {}
    for k in range(1, dim + 1):
        lower = {tuple(r): i for i, r in enumerate(by_dim[k - 1].tolist())}
        rows = by_dim[k].tolist()
        out = np.empty((len(rows), k + 1), dtype=np.int64)
        for i, row in enumerate(rows):
            for j in range(k + 1):
                out[i, j] = lower[tuple(row[:j] + row[j + 1:])]
        links[k] = out
    return by_dim, links


def delaunay(landmarks, seed: int = 0) -> Triangulation:
    """Del(L) in R^2 / R^3 with all faces and facet links (deterministic)."""
    pts = as_points(landmarks)
    dim = pts.shape[1]
    notes = []
    keep, dropped = _first_occurrences(pts)
    if dropped.size:
        notes.append(f"dropped {dropped.size} duplicate landmark(s)")
        pts = pts[keep]
    n = pts.shape[0]
    if n < dim + 1:
        raise DegeneracyError(f"need at least {dim + 1} distinct points in R^{dim}, got {n}")
    centered = pts - pts.mean(axis=0)
    tol = 1e-12 * max(1.0, float(np.abs(pts).max()))
    if int(np.linalg.matrix_rank(centered, tol=tol)) < dim:
        raise DegeneracyError("landmarks are affinely dependent (flat input)")

    scale = float(np.abs(pts).max()) or 1.0
    rng = np.random.Generator(np.random.Philox(seed))
    cells, jittered = None, False
    for attempt in range(4):
        if attempt == 0:
            work = pts
        else:
            noise = rng.uniform(-1.0, 1.0, size=pts.shape)
            work = pts + noise * JITTER_SCALE * scale * (10.0 ** (attempt - 1))
        try:
            got = _qhull_cells(work)
        except QhullError:
            continue
        # only the exact input is gated on general position; a jittered
        # input's qhull tie-break is already seeded and deterministic
        if attempt == 0 and _general_position_violated(
                work, np.sort(np.asarray(got, dtype=np.int64), axis=1)):
            continue
        cells = got
        if attempt > 0:
            jittered = True
            notes.append("input violates general position; applied seeded jitter "
                         f"(relative {JITTER_SCALE * 10.0 ** (attempt - 1):g})")
        break
    if cells is None:
        raise DegeneracyError("could not triangulate landmarks even after jitter")

    cells = np.sort(np.asarray(cells, dtype=np.int64), axis=1)
    by_dim, links = _close_faces(cells, dim)
    return Triangulation(dim=dim, points=pts, vertices=keep, simplices_by_dim=by_dim,
                         facet_links=links, dedup_dropped=dropped, jitter_applied=jittered,
                         warnings=tuple(notes))


def circumsphere_check(triangulation: Triangulation, tolerance: float = 1e-7) -> list:
    """(cell, landmark) pairs with the landmark deeper than `tolerance` inside
    the cell's circumsphere (empty list for a valid Delaunay complex)."""
    pts = triangulation.points
    cells = triangulation.top_cells
    centers, radii = circumcenters(pts, cells)
    bad = []
    for i, cell in enumerate(cells):
        if not np.isfinite(radii[i]):
            continue
        inside = np.flatnonzero(np.linalg.norm(pts - centers[i], axis=1) < radii[i] - tolerance)
        bad.extend((i, int(p)) for p in inside if p not in cell)
    return bad
