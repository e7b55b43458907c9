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
    """Circumcenter and radius of each full-dimensional cell (inf if flat).

    All cells at once: the (dim x dim) systems (e e^T) y = |e|^2 / 2 of the
    edge vectors e from each cell's first vertex are solved as one stacked
    LAPACK call; a singular (flat) cell gets center nan, radius inf.
    """
    dim = points.shape[1]
    n = cells.shape[0]
    centers = np.full((n, dim), np.nan)
    radii = np.full(n, np.inf)
    if n == 0:
        return centers, radii
    v = points[cells]                       # (n, dim + 1, dim)
    e = v[:, 1:, :] - v[:, :1, :]           # (n, dim, dim)
    rhs = 0.5 * np.einsum("nij,nij->ni", e, e)
    gram = e @ np.swapaxes(e, 1, 2)
    ok = np.ones(n, dtype=bool)
    try:
        y = np.linalg.solve(gram, rhs[..., None])[..., 0]
    except np.linalg.LinAlgError:  # some cell is flat: solve the rest one by one
        y = np.zeros((n, dim))
        for i in range(n):
            try:
                y[i] = np.linalg.solve(gram[i], rhs[i])
            except np.linalg.LinAlgError:
                ok[i] = False
    c = v[:, 0, :] + (y[:, None, :] @ e)[:, 0, :]
    centers[ok] = c[ok]
    radii[ok] = np.linalg.norm(c[ok] - v[ok, 0, :], axis=1)
    return centers, radii


def _general_position_violated(pts: np.ndarray, cells: np.ndarray) -> bool:
    """Some cell is flat, or its circumsphere (plus a 1e-9 relative slack)
    holds more than dim + 1 landmarks: the triangulation is then an
    arbitrary tie-break and the caller retries with a seeded jitter."""
    centers, radii = circumcenters(pts, cells)
    if not np.isfinite(radii).all():
        return True
    slack = GP_TOL * max(1.0, float(np.abs(pts).max()))
    counts = cKDTree(pts).query_ball_point(centers, radii + slack, return_length=True)
    return bool((np.asarray(counts) > pts.shape[1] + 1).any())


def _qhull_cells(work: np.ndarray):
    tri = _Qhull(work)
    if len(tri.coplanar):
        raise QhullError("qhull left coplanar points out of the triangulation")
    return tri.simplices


def _row_keys(rows: np.ndarray, base: int) -> np.ndarray:
    """Injective int64 key of each sorted vertex row (lexicographic order)."""
    key = np.zeros(rows.shape[0], dtype=np.int64)
    for j in range(rows.shape[1]):
        key = key * base + rows[:, j]
    return key


def _close_faces(cells: np.ndarray, dim: int):
    """Every face of the top cells, per dimension (sorted rows, lexicographic),
    and the facet links: links[k][i, j] = row in dimension k - 1 of simplex i
    without its j-th vertex."""
    base = int(cells.max()) + 1 if cells.size else 1
    by_dim = {}
    for k in range(dim + 1):
        if k == dim:
            faces = cells
        else:
            faces = np.concatenate([cells[:, list(c)] for c in combinations(range(dim + 1), k + 1)])
        # unique rows via their keys (a 1-D sort; key order = lexicographic)
        _, first = np.unique(_row_keys(faces, base), return_index=True)
        by_dim[k] = faces[first]
    links = {}
    for k in range(1, dim + 1):
        lower = _row_keys(by_dim[k - 1], base)  # ascending: rows are lexicographic
        rows = by_dim[k]
        out = np.empty((rows.shape[0], k + 1), dtype=np.int64)
        for j in range(k + 1):
            facet = np.delete(rows, j, axis=1)
            out[:, j] = np.searchsorted(lower, _row_keys(facet, base))
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
    tree = cKDTree(pts)
    for i in np.flatnonzero(np.isfinite(radii)):
        near = tree.query_ball_point(centers[i], max(radii[i] - tolerance, 0.0))
        for p in sorted(near):
            if p not in cells[i] and np.linalg.norm(pts[p] - centers[i]) < radii[i] - tolerance:
                bad.append((int(i), int(p)))
    return bad
