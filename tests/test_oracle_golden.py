"""Pin the CPU oracle (oracle/flood_oracle.c) to the reference's own outputs.

Golden fixtures were produced by running the reference
(tests/golden/make_golden.py); the oracle must reproduce them bit for bit.
"""

import numpy as np
import pytest

import oracle
from tests import _golden as G


@pytest.mark.parametrize("name", G.cases("fps"))
def test_oracle_fps_matches_reference(name):
    z = G.load("fps", name)
    got = oracle.fps(z["points"], int(z["k"]), int(z["start"]))
    np.testing.assert_array_equal(got, z["indices"])


@pytest.mark.parametrize("name", G.cases("flood"))
def test_oracle_flood_matches_reference(name):
    z = G.load("flood", name)
    sbd = G.simplices_by_dim(z)
    subset = str(z["landmark_mode"]) == "subset"
    got = oracle.flood_values(z["points"], z["tri_points"], sbd, int(z["grid_resolution"]),
                              subset_mode=subset)
    for k, want in G.values_by_dim(z).items():
        assert np.array_equal(np.sqrt(got[k]), want), f"dim {k}"


@pytest.mark.parametrize("name", ["rand3d_m4", "rand2d_m6", "dup3d_m5"])
def test_oracle_masking_invariance(name):
    """Lemma 4.2: masked values equal the unmasked definition (reference
    test_filtration.py::test_masking_invariance_against_unmasked)."""
    z = G.load("flood", name)
    sbd = G.simplices_by_dim(z)
    m = int(z["grid_resolution"])
    masked = oracle.flood_values(z["points"], z["tri_points"], sbd, m)
    for k in range(1, int(z["dim"]) + 1):
        un = oracle.unmasked_values(z["points"], z["tri_points"], sbd[k], m)
        assert np.array_equal(un, masked[k])


def test_oracle_skeleton_equals_full_complex():
    """Values of dims <= 2 do not depend on whether tetrahedra are top cells."""
    z = G.load("flood", "rand3d_m4")
    sbd = G.simplices_by_dim(z)
    full = oracle.flood_values(z["points"], z["tri_points"], sbd, 4)
    skel = oracle.flood_values(z["points"], z["tri_points"], sbd, 4, top_dim=2)
    for k in range(3):
        assert np.array_equal(full[k], skel[k])


def test_oracle_fps_thread_count_independent():
    rng = np.random.default_rng(5)
    pts = rng.random((20000, 3))
    a = oracle.fps(pts, 64, 3, threads=1)
    b = oracle.fps(pts, 64, 3, threads=7)
    np.testing.assert_array_equal(a, b)


def test_oracle_grid_matches_reference_embedding():
    from itertools import combinations

    rng = np.random.default_rng(3)
    verts = rng.normal(size=(4, 3))
    g = oracle.barycentric_grid(verts, 7)
    assert g.shape == (120, 3)  # C(10, 3)
    # rows of a face (zero weights elsewhere) equal the face's own grid bitwise
    g_face = oracle.barycentric_grid(verts[[0, 2]], 7)
    edge_rows = [r for r in g if any(np.array_equal(r, f) for f in g_face)]
    assert len(edge_rows) >= 8
    for i, j in combinations(range(4), 2):
        c, r = oracle.ritter(verts[[i, j]])
        np.testing.assert_allclose(r, np.linalg.norm(verts[i] - verts[j]) / 2, rtol=1e-15)
