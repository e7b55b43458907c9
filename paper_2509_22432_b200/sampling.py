"""The uniform-random sampler (reference floodph/filtration.py:303
_random_sampler_values), with the nearest-neighbour work on the GPU.

Per simplex the reference draws `sampler_count` flat-Dirichlet points from a
Philox generator seeded with (sampler_seed, k, row), prepends the simplex's
vertices, values the simplex by the largest exact nearest-neighbour distance
of those points, and completes it with its facets' values (monotone by
construction).  The draws stay on the host with the same numpy calls (the
sample coordinates must be bit-identical); the minimisation is one
fph_flood_samples call per dimension (the bounded-search kernel over the
explicit rows).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .geometry import sample_simplex_uniform


def _device_values(pts, tri, k, rows, samples, subset):
    lib = _native.require_gpu()
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    lms = np.ascontiguousarray(tri.points, dtype=np.float64)
    s4 = np.full((rows.shape[0], 4), -1, dtype=np.int32)
    s4[:, : k + 1] = rows
    smp = np.ascontiguousarray(samples, dtype=np.float64)
    out = np.empty(rows.shape[0])
    _native.check(lib.fph_flood_samples(
        _native.ptr(pts), pts.shape[0], pts.shape[1], _native.ptr(lms), lms.shape[0],
        _native.ptr(s4), rows.shape[0], k, _native.ptr(smp), smp.shape[1], 1 if subset else 0,
        _native.ptr(out), _native.FPH_MEM_HOST, None))
    return out


def random_sampler_values(pts, tri, config, subset: bool, top: int) -> dict:
    """{k: flood values of the k-simplices} under the uniform-random sampler."""
    values = {}
    nv = tri.simplices_by_dim[0].shape[0]
    if subset:
        values[0] = np.zeros(nv)
    else:
        verts = tri.simplices_by_dim[0]
        values[0] = np.sqrt(_device_values(pts, tri, 0, verts, tri.points[verts[:, 0]][:, None, :],
                                           False))
    count = int(config.sampler_count)
    for k in range(1, top + 1):
        rows = tri.simplices_by_dim[k]
        links = tri.facet_links[k]
        samples = np.empty((rows.shape[0], count + k + 1, tri.points.shape[1]))
        for i, row in enumerate(rows):
            verts = tri.points[row]
            samples[i, : k + 1] = verts
            samples[i, k + 1:] = sample_simplex_uniform(verts, count, seed=(config.sampler_seed, k, i))
        raw = np.sqrt(_device_values(pts, tri, k, rows, samples, subset)) if rows.shape[0] else np.zeros(0)
        values[k] = np.maximum(raw, values[k - 1][links].max(axis=1)) if rows.shape[0] else raw
    return values
