"""CPU oracle for the flood-filtration hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the CPU timing; the product package never does.

It wraps oracle/flood_oracle.c (a plain-C restatement of the reference's
algorithm, bit-exact in float64) through ctypes:

  fps(points, k, start)            reference floodph/geometry.py:88
  flood_values(points, tri, m)     reference floodph/filtration.py:233
                                   (_grid_values_masked: per top cell masked
                                   minimisation + face extraction, :227) and
                                   filtration.py:274 (external landmarks:
                                   exact nearest neighbour over the cloud)
  unmasked_values(...)             definition-level value per simplex

Pinned against the reference's own outputs in tests/golden (see
tests/golden/make_golden.py and tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from itertools import combinations

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libflood_oracle.so")
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.POINTER(ctypes.c_int64)
_i32 = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_fps.argtypes = [_d, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                              ctypes.c_int64, ctypes.c_int, _i64]
        L.orc_flood_cells.argtypes = [_d, ctypes.c_int64, ctypes.c_int, _d, _i64,
                                      ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                      _i64, _i32, _i64, ctypes.c_int, ctypes.c_int, _d]
        L.orc_flood_unmasked.argtypes = [_d, ctypes.c_int64, ctypes.c_int, _d, _i64,
                                         ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, _d]
        L.orc_barycentric_grid.argtypes = [ctypes.c_int, ctypes.c_int, _d, ctypes.c_int, _d]
        L.orc_ritter.argtypes = [_d, ctypes.c_int, ctypes.c_int, _d, _d]
        L.orc_grid_size.restype = ctypes.c_int64
        for f in ("orc_fps", "orc_flood_cells", "orc_flood_unmasked",
                  "orc_barycentric_grid", "orc_ritter"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


def fps(points, k: int, start: int = 0, threads: int = 0) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n, dim = pts.shape
    out = np.empty(k, dtype=np.int64)
    _check(lib().orc_fps(_ptr(pts, _d), n, dim, k, start, threads, _ptr(out, _i64)), "fps")
    return out


def barycentric_grid(verts, m: int) -> np.ndarray:
    v = np.ascontiguousarray(verts, dtype=np.float64)
    k = v.shape[0] - 1
    out = np.empty((int(lib().orc_grid_size(k, m)), v.shape[1]))
    _check(lib().orc_barycentric_grid(k, m, _ptr(v, _d), v.shape[1], _ptr(out, _d)), "grid")
    return out


def ritter(verts):
    v = np.ascontiguousarray(verts, dtype=np.float64)
    c = np.empty(v.shape[1])
    r = np.empty(1)
    _check(lib().orc_ritter(_ptr(v, _d), v.shape[0], v.shape[1], _ptr(c, _d), _ptr(r, _d)), "ritter")
    return c, float(r[0])


def face_owners(top_cells: np.ndarray, simplices_by_dim: dict):
    """CSR ownership: for each top cell, the faces it is the lex-first owner of.

    Mirrors reference floodph/filtration.py:198 _face_owners.  Returns
    (face_ptr, face_mask, face_out_dim, face_out_row).
    """
    kc = top_cells.shape[1] - 1
    row_index = {k: {tuple(r): i for i, r in enumerate(simplices_by_dim[k])} for k in range(kc + 1)}
    subsets = [S for size in range(1, kc + 2) for S in combinations(range(kc + 1), size)]
    ptr = [0]
    mask, out_dim, out_row = [], [], []
    seen = set()
    for cell in top_cells:
        t = tuple(int(v) for v in cell)
        for S in subsets:
            face = tuple(t[p] for p in S)
            if face in seen:
                continue
            seen.add(face)
            mask.append(sum(1 << p for p in S))
            out_dim.append(len(S) - 1)
            out_row.append(row_index[len(S) - 1][face])
        ptr.append(len(mask))
    return (np.asarray(ptr, np.int64), np.asarray(mask, np.int32),
            np.asarray(out_dim, np.int64), np.asarray(out_row, np.int64))


def flood_values(points, tri_points, simplices_by_dim: dict, m: int,
                 subset_mode: bool = True, threads: int = 0, top_dim=None) -> dict:
    """Squared flood values per dimension, {k: array aligned with simplices_by_dim[k]}.

    The reference algorithm: for each top cell, minimise over the masked
    candidates at every grid row, then give each owned face the max over its
    rows.  ``top_dim`` restricts the complex to its k-skeleton (cells = the
    k-simplices), which yields the same values for dims <= k.
    """
    X = np.ascontiguousarray(points, dtype=np.float64)
    tp = np.ascontiguousarray(tri_points, dtype=np.float64)
    kc = max(simplices_by_dim) if top_dim is None else top_dim
    cells = np.ascontiguousarray(simplices_by_dim[kc], dtype=np.int64)
    sub = {k: simplices_by_dim[k] for k in range(kc + 1)}
    ptr, mask, odim, orow = face_owners(cells, sub)
    offsets = np.zeros(kc + 2, dtype=np.int64)
    for k in range(kc + 1):
        offsets[k + 1] = offsets[k] + sub[k].shape[0]
    slots = np.ascontiguousarray(offsets[odim] + orow)
    out = np.full(int(offsets[-1]), np.nan)
    rc = lib().orc_flood_cells(
        _ptr(X, _d), X.shape[0], X.shape[1], _ptr(tp, _d), _ptr(cells, _i64),
        cells.shape[0], kc, m, _ptr(ptr, _i64), _ptr(mask, _i32), _ptr(slots, _i64),
        1 if subset_mode else 0, threads, _ptr(out, _d))
    _check(rc, "flood_cells")
    return {k: out[offsets[k]:offsets[k + 1]] for k in range(kc + 1)}


def unmasked_values(points, tri_points, simplices: np.ndarray, m: int, threads: int = 0) -> np.ndarray:
    """Squared value per simplex from the definition (whole cloud, own grid)."""
    X = np.ascontiguousarray(points, dtype=np.float64)
    tp = np.ascontiguousarray(tri_points, dtype=np.float64)
    s = np.ascontiguousarray(simplices, dtype=np.int64)
    out = np.empty(s.shape[0])
    _check(lib().orc_flood_unmasked(_ptr(X, _d), X.shape[0], X.shape[1], _ptr(tp, _d),
                                    _ptr(s, _i64), s.shape[0], s.shape[1] - 1, m, threads,
                                    _ptr(out, _d)), "unmasked")
    return out
