"""Build the pieces of a Triangulation from fixture arrays (tests only)."""

import numpy as np

from paper_2509_22432_b200.delaunay import Triangulation


def facet_links(by_dim):
    links = {}
    for k in range(1, max(by_dim) + 1):
        lower = {tuple(r): i for i, r in enumerate(by_dim[k - 1].tolist())}
        rows = by_dim[k].tolist()
        out = np.empty((len(rows), k + 1), dtype=np.int64)
        for i, row in enumerate(rows):
            for j in range(k + 1):
                out[i, j] = lower[tuple(row[:j] + row[j + 1:])]
        links[k] = out
    return links


def triangulation(points, by_dim):
    by_dim = {k: np.asarray(v, dtype=np.int64) for k, v in by_dim.items()}
    return Triangulation(dim=max(by_dim), points=np.asarray(points, dtype=np.float64),
                         vertices=np.arange(len(points)), simplices_by_dim=by_dim,
                         facet_links=facet_links(by_dim), dedup_dropped=np.zeros(0, np.int64),
                         jitter_applied=False, warnings=())


def sub_complex(by_dim, top_rows, top_dim):
    """Closure of the chosen top_dim simplices (rows into by_dim[top_dim])."""
    from itertools import combinations

    cells = by_dim[top_dim][np.asarray(top_rows)]
    out = {}
    for k in range(top_dim + 1):
        faces = np.concatenate([cells[:, list(c)] for c in combinations(range(top_dim + 1), k + 1)])
        out[k] = np.unique(faces, axis=0)
    return out
