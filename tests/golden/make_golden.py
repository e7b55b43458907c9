"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Each fixture stores the exact inputs and the
reference's outputs:

  fps_<name>.npz    points, k, start -> indices
                    (reference: floodph/geometry.py:88 farthest_point_sampling)
  flood_<name>.npz  points, landmark spec, grid_resolution -> triangulation
                    (tri.points, tri.vertices, simplices per dim) and the
                    flood value of every simplex per dim
                    (reference: floodph/filtration.py:348 build_flood_filtration,
                     masked-batch path filtration.py:233, kdtree path :274)
  sampler_<name>.npz  the same under the uniform-random sampler
                    (reference: floodph/filtration.py:303 _random_sampler_values)
  gap_<name>.npz    flood_value_exact_gap(simplex, m, X) pairs
                    (reference: floodph/filtration.py:178)
  mask_<name>.npz   compute_mask over a batch (CSR candidates) and
                    simplex_filtration of each cell's full grid
                    (reference: floodph/filtration.py:130, :165)
  diagram_<name>.npz  persistence bars of a reference FilteredComplex
                    (reference: floodph/persistence.py:49, :118)

The fixtures pin the CPU oracle (oracle/) and, through it, the CUDA path.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if not os.path.isdir(REF_SRC):
        raise SystemExit("reference sources not found; run in the build container")
    sys.path.insert(0, REF_SRC)
    import floodph  # noqa: F401

    return floodph


def _ref_digest() -> str:
    h = hashlib.sha256()
    for root, _, files in sorted(os.walk(REF_SRC)):
        for f in sorted(files):
            if f.endswith(".py"):
                with open(os.path.join(root, f), "rb") as fh:
                    h.update(fh.read())
    return h.hexdigest()[:16]


def fps_cases():
    from floodph.datagen import gen_circle, gen_torus

    yield "rand3d", np.random.default_rng(1).random((3000, 3)), 200, 0
    yield "rand2d", np.random.default_rng(2).random((5000, 2)), 300, 17
    yield "circle4096", gen_circle(4096).points, 12, 0
    yield "dup2d", np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 0.0], [1.0, 0.0]]), 4, 0
    yield "torus10k", gen_torus(10000, seed=0).points, 500, 0
    yield "k1", np.random.default_rng(0).random((10, 3)), 1, 7


def flood_cases():
    from floodph.datagen import gen_circle, gen_torus

    rng = np.random.default_rng
    yield "rand2d_m6", rng(10).random((600, 2)), 18, 6
    yield "rand3d_m4", rng(8).random((800, 3)), 25, 4
    yield "circle_m64", gen_circle(4096).points, 12, 64
    yield "rand3d_m1", rng(21).random((300, 3)), 10, 1
    yield "rand3d_m2", rng(22).random((300, 3)), 12, 2
    L = np.array([[0.0, 0.0], [8.0, 0.0], [4.0, 3.0]])
    yield "boundary2d", np.vstack([L, [[8.0, 4.0], [100.0, 100.0]]]), L, 8
    ext_x = rng(4).random((300, 2))
    ext_l = rng(4).random((15, 2)) + np.array([0.2, 0.1])
    yield "external2d", ext_x, ext_l, 8
    dup = rng(30).random((400, 3))
    yield "dup3d_m5", np.vstack([dup, dup[::7]]), 20, 5
    yield "rand3d_m30", rng(31).random((2000, 3)), 20, 30
    yield "torus10k_m20", gen_torus(10000, seed=0).points, 500, 20
    # reference acceptance criterion 2 (test_acceptance.py:99): X as its own
    # landmark set at m = 256, the first trials of its seeded sequence
    r202 = rng(202)
    for t in range(3):
        n = int(r202.integers(5, 11))
        X = r202.random((n, 2))
        yield f"accept2_m256_t{t}", X, X, 256
    # criterion 3 (test_acceptance.py:120): 10 FPS landmarks of 30 points
    X = rng(303).random((30, 2))
    from floodph.geometry import farthest_point_sampling

    yield "accept3_m256", X, X[farthest_point_sampling(X, 10)], 256
    yield "rand2d_m512", rng(40).random((300, 2)), 8, 512
    yield "rand3d_m300", rng(41).random((400, 3)), 6, 300


def sampler_cases():
    rng = np.random.default_rng
    yield "rand2d_c30", rng(13).random((400, 2)), 15, 30, 5
    yield "rand3d_c50", rng(14).random((600, 3)), 20, 50, 1
    ext_x = rng(15).random((300, 2))
    yield "external2d_c20", ext_x, rng(16).random((12, 2)) * 0.8 + 0.1, 20, 2


def gap_cases():
    rng = np.random.default_rng(12)  # reference test_filtration.py:262
    for i in range(5):
        verts = rng.random((3, 2)) * 2.0
        X = rng.random((60, 2)) * 2.0
        yield f"bracket{i}", verts, X, (16, 512)
    yield "unit_edge", np.array([[0.0, 0.0], [1.0, 0.0]]), np.array([[0.0, 0.0], [1.0, 0.0]]), (1,)
    yield "shrink", np.array([[0.0, 0.0], [2.0, 0.0], [0.5, 1.5]]), \
        np.array([[0.4, 0.2], [1.5, 0.3], [0.8, 1.0]]), (4, 8, 16, 32, 64)
    r = np.random.default_rng(13)
    X = r.random((500, 3))
    yield "tet_subset", X[[3, 77, 140, 402]], X, (6, 40)
    yield "tet_external", r.random((4, 3)) * 1.5 - 0.25, X, (5,)


def mask_cases():
    rng = np.random.default_rng
    X = rng(8).random((800, 3))
    yield "rand3d", X, 25, None
    # landmarks away from the cloud: empty balls fall back to the batch's
    # slab along the widest axis (x here), or to the whole cloud
    X = rng(51).random((400, 2)) * np.array([1.0, 0.5])
    yield "far2d_slab", X, None, np.array([[0.45, 3.0], [0.55, 3.0], [0.5, 3.1], [0.52, 3.3]])
    yield "far2d_cloud", X, None, np.array([[5.0, 3.0], [6.0, 3.0], [5.5, 4.0]])


def main() -> None:
    _ref()
    from floodph._kernels import warm_up
    from floodph.filtration import FloodConfig, build_flood_filtration
    from floodph.geometry import farthest_point_sampling

    warm_up()
    digest = _ref_digest()
    for name, pts, k, start in fps_cases():
        idx = farthest_point_sampling(pts, k, start=start)
        np.savez_compressed(
            os.path.join(OUT, f"fps_{name}.npz"),
            points=pts, k=k, start=start, indices=idx, ref_digest=digest,
        )
        print(f"fps_{name}: n={len(pts)} k={k}")
    for name, pts, L, count, seed in sampler_cases():
        cfg = FloodConfig(sampler="uniform-random", sampler_count=count, sampler_seed=seed,
                          threads=os.cpu_count())
        fc = build_flood_filtration(pts, L, cfg)
        tri = fc.meta["triangulation"]
        vm = fc.value_map()
        payload = dict(points=pts, sampler_count=count, sampler_seed=seed, tri_points=tri.points,
                       dim=tri.dim, landmark_mode=fc.meta["landmark_mode"], ref_digest=digest)
        if isinstance(L, (int, np.integer)):
            payload["n_landmarks"] = int(L)
        else:
            payload["landmarks"] = np.asarray(L, dtype=np.float64)
        for d in range(tri.dim + 1):
            rows = tri.simplices_by_dim[d]
            payload[f"simplices_{d}"] = rows
            payload[f"values_{d}"] = np.array([vm[tuple(int(v) for v in r)] for r in rows])
        np.savez_compressed(os.path.join(OUT, f"sampler_{name}.npz"), **payload)
        print(f"sampler_{name}: {tri.counts()}")
    from floodph.filtration import compute_mask, flood_value_exact_gap, simplex_filtration
    from floodph.geometry import barycentric_grid, barycentric_grid_template
    from floodph.persistence import boundary_matrix, reduce_and_extract
    from floodph.spatial import build_axis_sorted, widest_axis
    from floodph.delaunay import delaunay

    for name, verts, X, ms in gap_cases():
        vals = np.array([flood_value_exact_gap(verts, m, X) for m in ms])
        np.savez_compressed(os.path.join(OUT, f"gap_{name}.npz"), verts=verts, points=X,
                            ms=np.array(ms), values=vals, ref_digest=digest)
        print(f"gap_{name}: {vals.tolist()}")
    for name, X, nl, L in mask_cases():
        lm = X[farthest_point_sampling(X, nl)] if L is None else L
        tri = delaunay(lm)
        cells = tri.top_cells
        sc = build_axis_sorted(X, widest_axis(X))
        mask = compute_mask(tri, X, sc, cells)
        offs = np.concatenate([[0], np.cumsum([c.size for c in mask.candidates])])
        idx = np.concatenate(mask.candidates) if offs[-1] else np.zeros(0, np.int64)
        m = 5
        tpl = barycentric_grid_template(tri.dim, m)
        sf = np.array([simplex_filtration(tuple(c), barycentric_grid(tpl, tri.points[c]), cand, X)
                       for c, cand in zip(cells, mask.candidates)])
        np.savez_compressed(os.path.join(OUT, f"mask_{name}.npz"), points=X, tri_points=tri.points,
                            cells=cells, offsets=offs, indices=idx, axis=sc.axis, m=m,
                            simplex_values=sf, ref_digest=digest)
        print(f"mask_{name}: {cells.shape[0]} cells, {offs[-1]} candidates")
    for name, pts, L, m in flood_cases():
        t0 = time.time()
        cfg = FloodConfig(grid_resolution=m, threads=os.cpu_count())
        fc = build_flood_filtration(pts, L, cfg)
        tri = fc.meta["triangulation"]
        vm = fc.value_map()
        payload = dict(
            points=pts,
            grid_resolution=m,
            backend=fc.meta["backend"],
            landmark_mode=fc.meta["landmark_mode"],
            tri_points=tri.points,
            tri_vertices=tri.vertices,
            dim=tri.dim,
            ref_digest=digest,
        )
        if isinstance(L, (int, np.integer)):
            payload["n_landmarks"] = int(L)
            payload["landmark_indices"] = fc.meta["landmark_indices"]
        else:
            payload["landmarks"] = np.asarray(L, dtype=np.float64)
        for d in range(tri.dim + 1):
            rows = tri.simplices_by_dim[d]
            payload[f"simplices_{d}"] = rows
            payload[f"values_{d}"] = np.array([vm[tuple(int(v) for v in r)] for r in rows])
        np.savez_compressed(os.path.join(OUT, f"flood_{name}.npz"), **payload)
        print(f"flood_{name}: {tri.counts()} backend={fc.meta['backend']} {time.time() - t0:.1f}s")
        if name in ("torus10k_m20", "circle_m64", "rand3d_m4"):
            dgm = reduce_and_extract(boundary_matrix(fc), fc)
            bars = {f"bars_{k}": np.array(dgm.in_dim(k), dtype=np.float64).reshape(-1, 2)
                    for k in dgm.dimensions()}
            np.savez_compressed(os.path.join(OUT, f"diagram_{name}.npz"),
                                dims=np.array(dgm.dimensions()), ref_digest=digest, **bars)


if __name__ == "__main__":
    main()
