"""GPU: the rest of the reference's filtration API (floodph/filtration.py:88
CandidateMask, :130 compute_mask, :165 simplex_filtration, :178
flood_value_exact_gap) against golden vectors produced by running the
reference (tests/golden/make_golden.py).  Bit-exact."""

import numpy as np
import pytest

from paper_2509_22432_b200.delaunay import delaunay
from paper_2509_22432_b200.errors import IntegrityError
from paper_2509_22432_b200.filtration import (CandidateMask, compute_mask, flood_value_exact_gap,
                                              simplex_filtration)
from paper_2509_22432_b200.geometry import barycentric_grid, barycentric_grid_template
from paper_2509_22432_b200.spatial import build_axis_sorted
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", G.cases("gap"))
def test_exact_gap_golden(name):
    z = G.load("gap", name)
    for m, want in zip(z["ms"].tolist(), z["values"]):
        got = flood_value_exact_gap(z["verts"], int(m), z["points"])
        assert got == tuple(want), (m, got, tuple(want))


def test_exact_gap_contract():
    """Reference tests/test_filtration.py:258-284: the unit edge at m = 1,
    brackets shrinking with m, and the m = 512 value inside the m = 16
    bracket."""
    edge = np.array([[0.0, 0.0], [1.0, 0.0]])
    assert flood_value_exact_gap(edge, 1, edge) == (0.0, 1.0)
    verts = np.array([[0.0, 0.0], [2.0, 0.0], [0.5, 1.5]])
    X = np.array([[0.4, 0.2], [1.5, 0.3], [0.8, 1.0]])
    widths = [np.subtract(*flood_value_exact_gap(verts, m, X)[::-1]) for m in (4, 8, 16, 32, 64)]
    assert all(b < a for a, b in zip(widths, widths[1:]))
    rng = np.random.default_rng(12)
    for _ in range(5):
        v = rng.random((3, 2)) * 2.0
        Y = rng.random((60, 2)) * 2.0
        lo16, hi16 = flood_value_exact_gap(v, 16, Y)
        ref, _ = flood_value_exact_gap(v, 512, Y)
        assert lo16 <= ref + 1e-9 and ref <= hi16 + 1e-9
    with pytest.raises(ValueError):
        flood_value_exact_gap(edge, 0, edge)


@pytest.mark.parametrize("name", G.cases("mask"))
def test_compute_mask_and_simplex_filtration_golden(name):
    z = G.load("mask", name)
    X = z["points"]
    tri = delaunay(z["tri_points"])
    np.testing.assert_array_equal(tri.top_cells, z["cells"])
    sc = build_axis_sorted(X, int(z["axis"]))
    mask = compute_mask(tri, X, sc, z["cells"])
    assert isinstance(mask, CandidateMask)
    offs, idx = z["offsets"], z["indices"]
    assert len(mask.candidates) == z["cells"].shape[0]
    for i, cand in enumerate(mask.candidates):
        np.testing.assert_array_equal(cand, idx[offs[i]:offs[i + 1]])
    tpl = barycentric_grid_template(tri.dim, int(z["m"]))
    for c, cand, want in zip(z["cells"], mask.candidates, z["simplex_values"]):
        got = simplex_filtration(tuple(c), barycentric_grid(tpl, tri.points[c]), cand, X)
        assert got == want


def test_mask_edge_cases():
    z = G.load("mask", "rand3d")
    tri = delaunay(z["tri_points"])
    sc = build_axis_sorted(z["points"], 0)
    empty = compute_mask(tri, z["points"], sc, np.zeros((0, 4), np.int64))
    assert empty.candidates == []
    one = compute_mask(tri, z["points"], sc, z["cells"][0])  # a single row as 1-D
    assert len(one.candidates) == 1
    with pytest.raises(IntegrityError):
        simplex_filtration((0, 1), np.zeros((3, 3)), [], z["points"])
