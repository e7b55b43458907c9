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


def sampler_cases():
    rng = np.random.default_rng
    yield "rand2d_c30", rng(13).random((400, 2)), 15, 30, 5
    yield "rand3d_c50", rng(14).random((600, 3)), 20, 50, 1
    ext_x = rng(15).random((300, 2))
    yield "external2d_c20", ext_x, rng(16).random((12, 2)) * 0.8 + 0.1, 20, 2


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


if __name__ == "__main__":
    main()
