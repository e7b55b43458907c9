"""Host-side pieces of the path (no GPU): Delaunay policy against the
reference's complexes, the native persistence reduction against the Python
one, filtration order, config validation."""

import math

import numpy as np
import pytest

from paper_2509_22432_b200.delaunay import circumsphere_check, delaunay
from paper_2509_22432_b200.filtration import FilteredComplex, FloodConfig, filtration_order
from paper_2509_22432_b200.persistence import betti_at, boundary_matrix, reduce_and_extract
from tests import _complex as C
from tests import _golden as G


@pytest.mark.parametrize("name", G.cases("flood"))
def test_delaunay_matches_reference_complex(name):
    z = G.load("flood", name)
    if "landmark_indices" in z.files:
        lm = z["points"][z["landmark_indices"]]
    else:
        lm = z["landmarks"]
    tri = delaunay(lm)
    np.testing.assert_array_equal(tri.points, z["tri_points"])
    for k in range(int(z["dim"]) + 1):
        np.testing.assert_array_equal(tri.simplices_by_dim[k], z[f"simplices_{k}"])


def test_delaunay_square_needs_jitter():
    tri = delaunay(np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]))
    assert tri.counts() == {0: 4, 1: 5, 2: 2}
    assert tri.jitter_applied
    assert circumsphere_check(tri) == []


def _flood_complex(name):
    """A FilteredComplex of a golden case with its reference values."""
    z = G.load("flood", name)
    by_dim = G.simplices_by_dim(z)
    tri = C.triangulation(z["tri_points"], by_dim)
    values = G.values_by_dim(z)
    simplices = [(tuple(int(v) for v in r), k, float(values[k][i]))
                 for k in range(len(by_dim)) for i, r in enumerate(by_dim[k])]
    order = filtration_order(values, by_dim)
    return FilteredComplex(simplices=simplices, order=order, meta={"triangulation": tri})


@pytest.mark.parametrize("name", ["rand2d_m6", "rand3d_m4", "circle_m64", "torus10k_m20"])
def test_generic_and_triangulation_inputs_agree(name):
    """The same complex reduced from the triangulation's facet links and from
    a plain FilteredComplex (facets found by vertex lookup), with and without
    the clearing optimisation: identical diagrams."""
    fc = _flood_complex(name)
    plain = FilteredComplex(fc.simplices, fc.order, meta={})
    want = reduce_and_extract(boundary_matrix(fc), fc)
    for clearing in (True, False):
        assert reduce_and_extract(boundary_matrix(fc), fc, clearing=clearing).bars == want.bars
        assert reduce_and_extract(boundary_matrix(plain), plain, clearing=clearing).bars == want.bars


def test_filtration_order_matches_reference_sort():
    fc = _flood_complex("rand3d_m4")
    keys = [(v, d, verts) for verts, d, v in fc.simplices]
    ranks = sorted(range(len(keys)), key=lambda i: keys[i])
    want = np.empty(len(keys), dtype=np.int64)
    want[ranks] = np.arange(len(keys))
    np.testing.assert_array_equal(fc.order, want)


def test_reduction_hand_example():
    # triangle boundary, vertices at 0, edges at 1, 2, 3 (reference persistence tests)
    simplices = [((0,), 0, 0.0), ((1,), 0, 0.0), ((2,), 0, 0.0),
                 ((0, 1), 1, 1.0), ((0, 2), 1, 2.0), ((1, 2), 1, 3.0)]
    keys = [(v, d, s) for s, d, v in simplices]
    ranks = sorted(range(6), key=lambda i: keys[i])
    order = np.empty(6, dtype=np.int64)
    order[ranks] = np.arange(6)
    fc = FilteredComplex(simplices, order, meta={})
    dgm = reduce_and_extract(boundary_matrix(fc), fc)
    assert dgm.in_dim(0) == [(0.0, 1.0), (0.0, 2.0), (0.0, math.inf)]
    assert dgm.in_dim(1) == [(3.0, math.inf)]
    assert betti_at(dgm, 3.5, 1) == 1


def test_config_validation():
    for bad in (dict(grid_resolution=0), dict(batch_size=0), dict(sampler="sobol"),
                dict(backend="gpu"), dict(threads=0), dict(max_dim=4)):
        with pytest.raises(ValueError):
            FloodConfig(**bad).validate()
    FloodConfig(grid_resolution=512).validate()  # any m >= 1, as the reference
    FloodConfig(backend="kdtree").validate()


@pytest.mark.parametrize("name", G.cases("diagram"))
@pytest.mark.parametrize("clearing", [True, False])
def test_diagram_equals_reference_diagram(name, clearing):
    """The reference's own persistence diagram of its own values
    (tests/golden/diagram_*.npz from floodph.persistence): bars identical, so
    the bottleneck distance is 0 (the tolerance stated for diagrams is 0:
    values are bit-identical and the reduction is exact)."""
    fc = _flood_complex(name)
    dgm = reduce_and_extract(boundary_matrix(fc), fc, clearing=clearing)
    z = G.load("diagram", name)
    assert sorted(dgm.dimensions()) == sorted(int(d) for d in z["dims"])
    for d in z["dims"]:
        want = [tuple(b) for b in z[f"bars_{int(d)}"].tolist()]
        assert dgm.in_dim(int(d)) == want, int(d)


@pytest.mark.parametrize("name", ["rand3d_m4", "torus10k_m20"])
def test_lazy_columns_equal_reference_columns(name):
    """The flood-complex boundary matrix's lazily built columns equal the
    reference layout (sorted facet ranks, all below the column's rank)."""
    fc = _flood_complex(name)
    bm = boundary_matrix(fc)
    ranked = fc.in_order()
    rank_of = {v: j for j, (v, _, _) in enumerate(ranked)}
    from itertools import combinations

    for j, (verts, d, _) in enumerate(ranked):
        want = sorted(rank_of[f] for f in combinations(verts, d)) if d else []
        assert bm.columns[j] == want
        assert bm.dims[j] == d
    assert len(bm) == len(fc)


def test_face_order_violation_detected():
    fc = _flood_complex("rand2d_m6")
    order = fc.order.copy()
    # put an edge before one of its vertices
    e = next(i for i, s in enumerate(fc.simplices) if s[1] == 1)
    v = fc.simplices.index(next(s for s in fc.simplices if s[0] == (fc.simplices[e][0][0],)))
    order[e], order[v] = order[v], order[e]
    bad = FilteredComplex(fc.simplices, order, meta=fc.meta)
    from paper_2509_22432_b200.errors import IntegrityError

    with pytest.raises(IntegrityError):
        boundary_matrix(bad)


def test_missing_facet_detected():
    simplices = [((0,), 0, 0.0), ((1,), 0, 0.0), ((0, 1), 1, 1.0), ((0, 2), 1, 2.0)]
    fc = FilteredComplex(simplices, np.arange(4), meta={})
    from paper_2509_22432_b200.errors import IntegrityError

    with pytest.raises(IntegrityError, match="absent"):
        boundary_matrix(fc)


def test_generic_complex_not_grouped_by_dimension():
    """A user-built complex listing simplices out of dimension order reduces
    like the same complex grouped by dimension."""
    grouped = [((0,), 0, 0.0), ((1,), 0, 0.0), ((2,), 0, 0.0),
               ((0, 1), 1, 1.0), ((0, 2), 1, 2.0), ((1, 2), 1, 3.0), ((0, 1, 2), 2, 4.0)]
    shuffled = [grouped[i] for i in (3, 0, 6, 1, 5, 2, 4)]

    def fc_of(simplices):
        keys = [(v, d, s) for s, d, v in simplices]
        ranks = sorted(range(len(keys)), key=lambda i: keys[i])
        order = np.empty(len(keys), dtype=np.int64)
        order[ranks] = np.arange(len(keys))
        return FilteredComplex(simplices, order, meta={})

    a, b = fc_of(grouped), fc_of(shuffled)
    assert reduce_and_extract(boundary_matrix(a), a).bars == reduce_and_extract(boundary_matrix(b), b).bars
    assert reduce_and_extract(boundary_matrix(a), a).in_dim(1) == [(3.0, 4.0)]
