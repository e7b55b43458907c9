"""GPU parity at the BASELINE.json configs' full sizes, against the CPU
oracle (oracle/, pinned to the reference's goldens).  Landmark indices must
be identical; flood values bit-identical (tolerance 0).

  configs[1]  1M sphere+torus, 2k landmarks, dims <= 2, m = 20: FPS and the
              COMPLETE complex (every triangle, edge and vertex)
  configs[4]  the same cloud at m = 30: 6000 random triangles with faces
  configs[2]  10M uniform box, 5k landmarks, full tetrahedra: FPS (tiled
              kernel) and 300 random tetrahedra with all their faces
  configs[3]  batch of ModelNet-shaped 100k clouds, 1k landmarks: batched
              FPS of a 64-cloud batch, and 3 of its clouds' full complexes

Reference paths: floodph/geometry.py:88 (FPS), floodph/filtration.py:233-271
(the masked flood values)."""

import numpy as np
import pytest

import oracle
from paper_2509_22432_b200 import farthest_point_sampling, farthest_point_sampling_batched
from paper_2509_22432_b200.datagen import (gen_modelnet_batch, gen_sphere_torus_mix,
                                           gen_uniform_box)
from paper_2509_22432_b200.delaunay import delaunay
from paper_2509_22432_b200.filtration import flood_sq_values
from tests import _complex as C

pytestmark = pytest.mark.gpu


def _sample_check(X, tri, sq, top, m, n_top, seed):
    """n_top random top simplices + all their faces against the oracle."""
    rows = np.random.default_rng(seed).choice(tri.simplices_by_dim[top].shape[0],
                                              min(n_top, tri.simplices_by_dim[top].shape[0]),
                                              replace=False)
    sub = C.sub_complex(tri.simplices_by_dim, rows, top)
    want = oracle.flood_values(X, tri.points, sub, m, top_dim=top)
    for k in range(1, top + 1):
        index = {tuple(r): i for i, r in enumerate(tri.simplices_by_dim[k].tolist())}
        got = np.array([sq[k][index[tuple(r)]] for r in sub[k].tolist()])
        assert np.array_equal(got, want[k]), k
    return sum(v.shape[0] for v in sub.values())


@pytest.fixture(scope="module")
def sphere_torus_1m():
    X = gen_sphere_torus_mix(1_000_000, seed=0).points
    idx = farthest_point_sampling(X, 2000)
    return X, idx, delaunay(X[idx])


def test_configs1_fps_matches_oracle(sphere_torus_1m):
    X, idx, _ = sphere_torus_1m
    np.testing.assert_array_equal(idx, oracle.fps(X, 2000, 0))


def test_configs1_complete_complex_matches_oracle(sphere_torus_1m):
    """Every simplex of dim <= 2 of the configs[1] complex (40k simplices)."""
    X, _, tri = sphere_torus_1m
    sq = flood_sq_values(X, tri, 20, True, 2)
    want = oracle.flood_values(X, tri.points, {k: tri.simplices_by_dim[k] for k in range(3)}, 20,
                               top_dim=2)
    for k in range(3):
        assert np.array_equal(sq[k], want[k]), k


def test_configs4_dense_m30_matches_oracle(sphere_torus_1m):
    X, _, tri = sphere_torus_1m
    sq = flood_sq_values(X, tri, 30, True, 2)
    for k in range(3):
        assert np.isfinite(sq[k]).all()
    assert (sq[1][tri.facet_links[2]] <= sq[2][:, None]).all()
    _sample_check(X, tri, sq, 2, 30, 6000, seed=4)


@pytest.fixture(scope="module")
def box_10m():
    X = gen_uniform_box(10_000_000, seed=0).points
    idx = farthest_point_sampling(X, 5000)
    return X, idx


def test_configs2_fps_10m_matches_oracle(box_10m):
    X, idx = box_10m
    np.testing.assert_array_equal(idx, oracle.fps(X, 5000, 0))


def test_configs2_tetrahedra_match_oracle(box_10m):
    X, idx = box_10m
    tri = delaunay(X[idx])
    assert tri.dim == 3
    sq = flood_sq_values(X, tri, 20, True, 3)
    for k in range(1, 4):
        assert (sq[k - 1][tri.facet_links[k]] <= sq[k][:, None]).all()
    _sample_check(X, tri, sq, 3, 20, 300, seed=2)


def test_configs3_batch_fps_and_clouds_match_oracle():
    clouds = gen_modelnet_batch(64, 100_000, seed=0)
    got = farthest_point_sampling_batched(clouds, 1000, 0)
    for b in (0, 31, 63):
        np.testing.assert_array_equal(got[b], oracle.fps(clouds[b], 1000, 0))
        X = clouds[b]
        tri = delaunay(X[got[b]])
        sq = flood_sq_values(X, tri, 20, True)
        want = oracle.flood_values(X, tri.points, tri.simplices_by_dim, 20)
        for k in range(tri.dim + 1):
            assert np.array_equal(sq[k], want[k]), (b, k)
