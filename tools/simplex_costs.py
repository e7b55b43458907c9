"""Per-simplex cost anatomy of the bounded search on configs[1] triangles:
cycles per phase vs candidate count (debug capture of fph_flood_interior)."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2509_22432_b200 import _native, farthest_point_sampling
    from paper_2509_22432_b200.datagen import gen_sphere_torus_mix
    from paper_2509_22432_b200.delaunay import delaunay

    lib = _native.require_gpu()
    X = gen_sphere_torus_mix(1_000_000, seed=0).points
    tri = delaunay(X[farthest_point_sampling(X, 2000)])
    lms = np.ascontiguousarray(tri.points)
    out = {}
    for k in (1, 2):
        rows = tri.simplices_by_dim[k]
        s4 = np.full((rows.shape[0], 4), -1, dtype=np.int32)
        s4[:, : k + 1] = rows
        sq = np.empty(rows.shape[0])
        lib.fph_debug_simplex_cycles(1, None, 0, None)
        _native.check(lib.fph_flood_interior(_native.ptr(X), X.shape[0], 3, _native.ptr(lms), lms.shape[0],
                                             _native.ptr(s4), rows.shape[0], k, 20, 1, _native.ptr(sq),
                                             _native.FPH_MEM_HOST, None))
        buf = np.empty(8 * rows.shape[0], dtype=np.int64)
        n = np.zeros(1, dtype=np.int64)
        lib.fph_debug_simplex_cycles(0, buf.ctypes.data, buf.size, n.ctypes.data)
        d = buf.reshape(-1, 8)
        # candidate counts from the Ritter balls (host, for binning)
        V = tri.points[rows]
        best = np.full(len(rows), -1.0)
        c = np.zeros((len(rows), 3))
        for i in range(k + 1):
            for j in range(i + 1, k + 1):
                dd = ((V[:, i] - V[:, j]) ** 2).sum(1)
                u = dd > best
                best[u] = dd[u]
                c[u] = 0.5 * (V[u, i] + V[u, j])
        from scipy.spatial import cKDTree

        r = np.sqrt(((V - c[:, None]) ** 2).sum(2).max(1))
        C = cKDTree(X).query_ball_point(c, np.sqrt(2) * r, return_length=True)
        tot = d[:, :4].sum(1).astype(float)
        edges = [0, 512, 2000, 5000, 20000, 50000, 131072, 10 ** 9]
        rep = []
        for lo, hi in zip(edges[:-1], edges[1:]):
            m = (C > lo) & (C <= hi)
            if m.any():
                team = d[m, 7] > 1
                rep.append({"C": f"({lo},{hi}]", "n": int(m.sum()),
                            "cycles_share": float(tot[m].sum() / tot.sum()),
                            "warp_cycles_mean": float(tot[m].mean()),
                            "phase_share": [float(d[m, i].sum() / max(tot[m].sum(), 1)) for i in range(4)],
                            "blocks_searched_mean": float(d[m, 4].mean()),
                            "blocks_pruned_mean": float(d[m, 5].mean()),
                            "staged_mean": float(d[m, 6].mean()), "team": int(team.sum())})
        out[f"dim{k}"] = rep
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
