"""GPU parity: the CUDA path through the C ABI against the reference's golden
vectors and the CPU oracle.  Integer outputs (landmark indices) must be
identical; float64 flood values must be bit-identical (tolerance 0, stricter
than the north star's 1e-5 relative fp32 bar)."""

import numpy as np
import pytest

import oracle
from paper_2509_22432_b200 import farthest_point_sampling, farthest_point_sampling_batched
from paper_2509_22432_b200.datagen import gen_sphere_torus_mix, gen_torus
from paper_2509_22432_b200.delaunay import delaunay
from paper_2509_22432_b200.filtration import FloodConfig, build_flood_filtration, flood_sq_values
from tests import _complex as C
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", G.cases("fps"))
def test_fps_golden(name):
    z = G.load("fps", name)
    got = farthest_point_sampling(z["points"], int(z["k"]), int(z["start"]))
    np.testing.assert_array_equal(got, z["indices"])


@pytest.mark.parametrize("n,dim,k,start", [(200_000, 3, 300, 0), (50_001, 2, 500, 123),
                                           (1_500_000, 3, 40, 7), (3, 2, 3, 2)])
def test_fps_matches_oracle(n, dim, k, start):
    pts = np.random.default_rng(n).random((n, dim))
    got = farthest_point_sampling(pts, k, start)
    np.testing.assert_array_equal(got, oracle.fps(pts, k, start))


@pytest.mark.parametrize("n,dim,k,start", [(2_000_000, 3, 300, 5), (1_400_000, 2, 200, 0)])
def test_fps_tiled_matches_oracle(n, dim, k, start):
    """Clouds beyond shared-memory residency take the Morton-tiled kernel."""
    pts = np.random.default_rng(n + 1).normal(size=(n, dim))
    got = farthest_point_sampling(pts, k, start)
    np.testing.assert_array_equal(got, oracle.fps(pts, k, start))


def test_fps_tiled_lattice_ties():
    g = np.stack(np.meshgrid(np.arange(120.0), np.arange(120.0), np.arange(100.0)), -1).reshape(-1, 3)
    got = farthest_point_sampling(g, 150, 17)
    np.testing.assert_array_equal(got, oracle.fps(g, 150, 17))


@pytest.mark.parametrize("batch,n,k", [(20, 100_000, 64), (7, 3_000, 200), (3, 200_000, 16)])
def test_fps_batched_matches_oracle(batch, n, k):
    from paper_2509_22432_b200 import farthest_point_sampling_batched

    clouds = np.random.default_rng(batch * n).random((batch, n, 3))
    got = farthest_point_sampling_batched(clouds, k, 3)
    for b in range(batch):
        np.testing.assert_array_equal(got[b], oracle.fps(clouds[b], k, 3))


_RES_NT = 512  # threads per CTA of the resident / batched FPS kernels (csrc/fph_fps.cu kResNT)


@pytest.mark.parametrize("pt", list(range(1, 19)))
def test_fps_resident_points_per_thread(pt):
    """Every PT instantiation of the resident kernel (slices of PT x 512
    points per CTA, padded): n chosen from the device's SM count so the
    slice needs exactly PT points per thread, with a ragged last slice;
    coordinates quantised to 1/8 so ties are common."""
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = sms * (pt * _RES_NT - 100) + 37
    pts = np.round(np.random.default_rng(pt).random((n, 3)) * 64) / 8
    got = farthest_point_sampling(pts, 120, pt)
    np.testing.assert_array_equal(got, oracle.fps(pts, 120, pt))


@pytest.mark.parametrize("pt", list(range(1, 19)))
def test_fps_batched_points_per_thread(pt):
    """Every PT instantiation of the batched kernel (one CTA per cloud up to
    9216 points): clouds of PT x 512 - 100 points, quantised coordinates."""
    n = pt * _RES_NT - 100
    clouds = np.round(np.random.default_rng(100 + pt).random((5, n, 3)) * 64) / 8
    got = farthest_point_sampling_batched(clouds, 50, 1)
    for b in range(5):
        np.testing.assert_array_equal(got[b], oracle.fps(clouds[b], 50, 1))


def test_fps_ties_uniform_grid():
    # a lattice is full of exact ties: lowest index must win every time
    g = np.stack(np.meshgrid(np.arange(40.0), np.arange(40.0), np.arange(5.0)), -1).reshape(-1, 3)
    got = farthest_point_sampling(g, 200, 0)
    np.testing.assert_array_equal(got, oracle.fps(g, 200, 0))


@pytest.mark.parametrize("name", G.cases("flood"))
def test_flood_values_golden(name):
    z = G.load("flood", name)
    tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
    subset = str(z["landmark_mode"]) == "subset"
    sq = flood_sq_values(z["points"], tri, int(z["grid_resolution"]), subset)
    for k, want in G.values_by_dim(z).items():
        got = np.sqrt(sq[k])
        assert np.array_equal(got, want), (k, np.abs(got - want).max())


@pytest.mark.parametrize("name", G.cases("flood"))
def test_build_flood_filtration_golden(name):
    """End to end through the drop-in API: same complex, same values."""
    z = G.load("flood", name)
    m = int(z["grid_resolution"])
    L = int(z["n_landmarks"]) if "n_landmarks" in z.files else z["landmarks"]
    fc = build_flood_filtration(z["points"], L, FloodConfig(grid_resolution=m))
    tri = fc.meta["triangulation"]
    for k, want in G.values_by_dim(z).items():
        np.testing.assert_array_equal(tri.simplices_by_dim[k], z[f"simplices_{k}"])
    vm = fc.value_map()
    for k, want in G.values_by_dim(z).items():
        got = np.array([vm[tuple(int(v) for v in r)] for r in z[f"simplices_{k}"]])
        assert np.array_equal(got, want)
    if "landmark_indices" in z.files:
        np.testing.assert_array_equal(fc.meta["landmark_indices"], z["landmark_indices"])


@pytest.mark.parametrize("n,nl,m,max_dim", [(100_000, 300, 8, 3), (60_000, 400, 20, 2),
                                            (30_000, 150, 30, 1)])
def test_flood_matches_oracle_mid_size(n, nl, m, max_dim):
    X = gen_sphere_torus_mix(n, seed=n).points
    idx = farthest_point_sampling(X, nl)
    tri = delaunay(X[idx])
    sq = flood_sq_values(X, tri, m, True, max_dim)
    want = oracle.flood_values(X, tri.points, {k: tri.simplices_by_dim[k] for k in range(max_dim + 1)},
                               m, top_dim=max_dim)
    for k in range(max_dim + 1):
        assert np.array_equal(sq[k], want[k]), k


def test_flood_external_landmarks_mid_size():
    rng = np.random.default_rng(9)
    X = rng.random((20_000, 3))
    L = rng.random((60, 3)) * 1.2 - 0.1
    fc = build_flood_filtration(X, L, FloodConfig(grid_resolution=5))
    assert fc.meta["landmark_mode"] == "external"
    tri = fc.meta["triangulation"]
    want = oracle.flood_values(X, tri.points, tri.simplices_by_dim, 5, subset_mode=False)
    vm = fc.value_map()
    for k in range(4):
        got = np.array([vm[tuple(int(v) for v in r)] for r in tri.simplices_by_dim[k]])
        assert np.array_equal(got, np.sqrt(want[k]))


def test_flood_full_size_properties_and_sampled_oracle():
    """BASELINE configs[1] size: 1M sphere+torus, 2k landmarks, dims <= 2.
    Checked: idempotence, monotonicity, vertices 0, and a random sample of
    triangles (with their edges) against the oracle bit for bit."""
    X = gen_sphere_torus_mix(1_000_000, seed=0).points
    idx = farthest_point_sampling(X, 2000)
    tri = delaunay(X[idx])
    sq1 = flood_sq_values(X, tri, 20, True, 2)
    sq2 = flood_sq_values(X, tri, 20, True, 2)
    for k in range(3):
        assert np.array_equal(sq1[k], sq2[k])
        assert np.isfinite(sq1[k]).all() and (sq1[k] >= 0).all()
    assert (sq1[0] == 0).all()
    for k in (1, 2):
        assert (sq1[k - 1][tri.facet_links[k]] <= sq1[k][:, None]).all()
    rng = np.random.default_rng(0)
    rows = rng.choice(tri.simplices_by_dim[2].shape[0], 48, replace=False)
    sub = C.sub_complex(tri.simplices_by_dim, rows, 2)
    want = oracle.flood_values(X, tri.points, sub, 20, top_dim=2)
    for k in (1, 2):
        index = {tuple(r): i for i, r in enumerate(tri.simplices_by_dim[k].tolist())}
        got = np.array([sq1[k][index[tuple(r)]] for r in sub[k].tolist()])
        assert np.array_equal(got, want[k]), k


@pytest.fixture
def algo_switch():
    from paper_2509_22432_b200 import _native

    lib = _native.require_gpu()

    def use(algo, reps=0, team=0):
        _native.check(lib.fph_set_search(algo, reps, team))

    yield use
    use(1)


@pytest.mark.parametrize("reps,team", [(1024, 32768), (64, 1000), (4096, 2**30), (300, 1),
                                       (512, 0), (512, -50)])
def test_block_search_equals_brute_force_full_size(algo_switch, reps, team):
    """The two exact algorithms agree bit for bit on BASELINE configs[1]
    (1M points, 2k landmarks, dims <= 2) for several search tunings: sample
    sizes, and every simplex searched by one warp / by a whole CTA / by the
    device-derived team threshold (team <= 0)."""
    X = gen_sphere_torus_mix(1_000_000, seed=0).points
    tri = delaunay(X[farthest_point_sampling(X, 2000)])
    algo_switch(0)
    brute = flood_sq_values(X, tri, 20, True, 2)
    algo_switch(1, reps, team)
    search = flood_sq_values(X, tri, 20, True, 2)
    for k in range(3):
        assert np.array_equal(brute[k], search[k]), k


@pytest.mark.parametrize("algo,reps,team", [(0, 0, 0), (1, 0, 0), (1, 16, 1), (1, 16, 2**30)])
@pytest.mark.parametrize("name", ["torus10k_m20", "rand3d_m30", "external2d", "circle_m64",
                                  "dup3d_m5"])
def test_both_algorithms_golden(algo_switch, algo, reps, team, name):
    algo_switch(algo, reps, team)
    z = G.load("flood", name)
    tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
    subset = str(z["landmark_mode"]) == "subset"
    sq = flood_sq_values(z["points"], tri, int(z["grid_resolution"]), subset)
    for k, want in G.values_by_dim(z).items():
        assert np.array_equal(np.sqrt(sq[k]), want), k


@pytest.mark.parametrize("team", [0, 1, 2**30])
@pytest.mark.parametrize("name", G.cases("flood"))
def test_phase_kernel_chain_golden(algo_switch, monkeypatch, team, name):
    """The four phase kernels chained per simplex (PDL + stage flags; the
    default for complexes >= 10 000 simplices) forced onto every golden
    complex, with warp-only, CTA-team-only and auto team scheduling."""
    monkeypatch.setenv("FPH_SPLIT_MIN_SIMPLICES", "0")
    algo_switch(1, 0, team)
    z = G.load("flood", name)
    tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
    subset = str(z["landmark_mode"]) == "subset"
    sq = flood_sq_values(z["points"], tri, int(z["grid_resolution"]), subset)
    for k, want in G.values_by_dim(z).items():
        assert np.array_equal(np.sqrt(sq[k]), want), k


@pytest.mark.parametrize("name", G.cases("sampler"))
def test_uniform_random_sampler_golden(name):
    """Reference uniform-random sampler (filtration.py:303): same Philox draws
    on the host, nearest neighbours on the GPU; values within 1e-12 relative
    (the reference takes cKDTree's neighbour, exact up to distance ties)."""
    z = G.load("sampler", name)
    L = int(z["n_landmarks"]) if "n_landmarks" in z.files else z["landmarks"]
    cfg = FloodConfig(sampler="uniform-random", sampler_count=int(z["sampler_count"]),
                      sampler_seed=int(z["sampler_seed"]))
    fc = build_flood_filtration(z["points"], L, cfg)
    vm = fc.value_map()
    assert fc.meta["landmark_mode"] == str(z["landmark_mode"])
    for k in range(int(z["dim"]) + 1):
        got = np.array([vm[tuple(int(v) for v in r)] for r in z[f"simplices_{k}"]])
        np.testing.assert_allclose(got, z[f"values_{k}"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_values_equal_single_gpu(world):
    """Every rank's share (computed here one rank after another on one GPU,
    no collective) reassembled and completed equals the single-call values."""
    import torch

    from paper_2509_22432_b200.parallel import complete, shard_interior

    X = gen_sphere_torus_mix(200_000, seed=3).points
    tri = delaunay(X[farthest_point_sampling(X, 500)])
    want = flood_sq_values(X, tri, 12, True, 3)
    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    lm = torch.from_numpy(np.ascontiguousarray(tri.points)).to(dev)
    by_dim = {k: torch.from_numpy(np.ascontiguousarray(tri.simplices_by_dim[k], dtype=np.int32)).to(dev)
              for k in range(4)}
    fac = {k: torch.from_numpy(np.ascontiguousarray(tri.facet_links[k], dtype=np.int32)).to(dev)
           for k in range(1, 4)}
    shares = [shard_interior(Xd, lm, by_dim, 3, 12, True, r, world) for r in range(world)]
    interior = {}
    for k in range(1, 4):
        full = torch.empty(by_dim[k].shape[0], dtype=torch.float64, device=dev)
        for r in range(world):
            full[r::world] = shares[r][k]
        interior[k] = full
    got = complete(interior, fac, by_dim[0].shape[0], 3, True)
    for k in range(4):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k


# ------------------------------------------------------------- edge cases
def test_empty_and_tiny_inputs():
    from paper_2509_22432_b200 import _native

    lib = _native.require_gpu()
    X = np.random.default_rng(0).random((50, 3))
    lm = X[:5].copy()
    # zero simplices: nothing to do, success
    out = np.empty(1)
    _native.check(lib.fph_flood_interior(_native.ptr(X), 50, 3, _native.ptr(lm), 5,
                                         _native.ptr(np.zeros((1, 4), np.int32)), 0, 2, 8, 1,
                                         _native.ptr(out), _native.FPH_MEM_HOST, None))
    # single-point cloud FPS, k = 1
    np.testing.assert_array_equal(farthest_point_sampling(np.array([[0.5, 0.5]]), 1, 0), [0])
    with pytest.raises(ValueError):
        farthest_point_sampling(np.array([[0.5, 0.5]]), 2, 0)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_low_resolution_has_no_interior_rows(m):
    """m <= k: a k-simplex has no interior rows; its value comes from its
    facets alone (reference: grid = vertices and edge points only)."""
    z = G.load("flood", "rand3d_m1") if m == 1 else G.load("flood", "rand3d_m2")
    X = z["points"]
    tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
    sq = flood_sq_values(X, tri, m, True)
    want = oracle.flood_values(X, tri.points, tri.simplices_by_dim, m)
    for k in range(4):
        assert np.array_equal(sq[k], want[k])


def test_planar_cloud_full_size_sampled_oracle():
    """2-D cloud (z = 0 internally): 500k noisy circle-annulus points."""
    rng = np.random.default_rng(3)
    th = rng.uniform(0, 2 * np.pi, 500_000)
    r = 1.0 + 0.02 * rng.normal(size=th.size)
    X = np.c_[r * np.cos(th), r * np.sin(th)]
    tri = delaunay(X[farthest_point_sampling(X, 300)])
    sq = flood_sq_values(X, tri, 16, True)
    rows = np.random.default_rng(1).choice(tri.simplices_by_dim[2].shape[0], 40, replace=False)
    sub = C.sub_complex(tri.simplices_by_dim, rows, 2)
    want = oracle.flood_values(X, tri.points, sub, 16, top_dim=2)
    for k in (1, 2):
        index = {tuple(rw): i for i, rw in enumerate(tri.simplices_by_dim[k].tolist())}
        got = np.array([sq[k][index[tuple(rw)]] for rw in sub[k].tolist()])
        assert np.array_equal(got, want[k])


def test_duplicate_points_and_landmarks():
    """Duplicates in the cloud; FPS beyond the distinct count picks
    duplicates (value 0 rows); Delaunay drops duplicate landmarks."""
    rng = np.random.default_rng(5)
    base = rng.random((200, 3))
    X = np.vstack([base, base])
    idx = farthest_point_sampling(X, 300)
    np.testing.assert_array_equal(idx, oracle.fps(X, 300))
    fc = build_flood_filtration(X, 250, FloodConfig(grid_resolution=4))
    tri = fc.meta["triangulation"]
    assert tri.dedup_dropped.size == 50
    want = oracle.flood_values(X, tri.points, tri.simplices_by_dim, 4)
    vm = fc.value_map()
    for k in range(4):
        got = np.array([vm[tuple(int(v) for v in r)] for r in tri.simplices_by_dim[k]])
        assert np.array_equal(got, np.sqrt(want[k]))


@pytest.mark.parametrize("m", [255, 256, 257, 700])
def test_high_resolutions_match_oracle(algo_switch, m):
    """Resolutions past one byte (template rows are ushort4; the weight
    table grows with m) under both algorithms."""
    z = G.load("flood", "rand2d_m6")
    tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
    want = oracle.flood_values(z["points"], tri.points, tri.simplices_by_dim, m)
    for algo in (0, 1):
        algo_switch(algo)
        sq = flood_sq_values(z["points"], tri, m, True)
        for k in range(3):
            assert np.array_equal(sq[k], want[k]), (algo, k)


def test_bad_resolutions():
    z = G.load("flood", "rand2d_m6")
    tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
    for m in (0, -3, 65536):
        with pytest.raises(ValueError):
            flood_sq_values(z["points"], tri, m, True)
    with pytest.raises(ValueError):  # C(m - 1, 3) interior rows per tetrahedron >= 2^24
        z3 = G.load("flood", "rand3d_m4")
        flood_sq_values(z3["points"], C.triangulation(z3["tri_points"], G.simplices_by_dim(z3)),
                        2000, True)


# ------------------------------------------------- pipeline acceptance
def test_circle_golden_diagram():
    """Reference acceptance criterion 1 (Appendix circle example): 4096
    uniform-angle circle points, 12 FPS landmarks, m = 64: H0 deaths
    1 - cos(pi/16) x 8 and 1 - cos(pi/8) x 3 plus one essential bar; one H1
    bar (1 - cos(pi/8), 1); tolerance 2e-3."""
    import math

    from paper_2509_22432_b200 import flood_diagram
    from paper_2509_22432_b200.datagen import gen_circle

    dgm, fc = flood_diagram(gen_circle(4096), 12, FloodConfig(grid_resolution=64))
    short, long_ = 1 - math.cos(math.pi / 16), 1 - math.cos(math.pi / 8)
    h0 = dgm.in_dim(0)
    deaths = [d for _, d in h0]
    assert len(h0) == 12 and all(b == 0.0 for b, _ in h0)
    assert sum(abs(d - short) < 2e-3 for d in deaths) == 8
    assert sum(abs(d - long_) < 2e-3 for d in deaths) == 3
    assert sum(math.isinf(d) for d in deaths) == 1
    h1 = dgm.in_dim(1)
    assert len(h1) == 1 and abs(h1[0][0] - long_) < 2e-3 and abs(h1[0][1] - 1.0) < 2e-3


def test_torus_topology_and_reference_diagram():
    """configs[0] (10k torus points, 500 landmarks, m = 20): the diagram
    equals the one computed from the reference's own values (golden), and
    the torus shows Betti (1, 2, 1) at a mid radius."""
    from paper_2509_22432_b200 import flood_diagram
    from paper_2509_22432_b200.persistence import betti_at

    z = G.load("flood", "torus10k_m20")
    dgm, fc = flood_diagram(z["points"], 500, FloodConfig(grid_resolution=20))
    # rebuild the complex with the reference values: same diagram
    from paper_2509_22432_b200.filtration import FilteredComplex, filtration_order
    from paper_2509_22432_b200.persistence import boundary_matrix, reduce_and_extract

    vals = G.values_by_dim(z)
    by_dim = G.simplices_by_dim(z)
    simplices = [(tuple(int(v) for v in r), k, float(vals[k][i]))
                 for k in range(4) for i, r in enumerate(by_dim[k])]
    ref_fc = FilteredComplex(simplices, filtration_order(vals, by_dim),
                             meta={"triangulation": fc.meta["triangulation"]})
    ref_dgm = reduce_and_extract(boundary_matrix(ref_fc), ref_fc)
    assert dgm.bars == ref_dgm.bars
    r = 0.3
    assert (betti_at(dgm, r, 0), betti_at(dgm, r, 1), betti_at(dgm, r, 2)) == (1, 2, 1)


# ------------------------------------------------- adversarial numerics
@pytest.mark.parametrize("scale,offset", [(1.0, 1e4), (1e-6, 0.0), (1e6, 3e6), (1.0, -7.5e2)])
def test_scaled_and_offset_clouds(algo_switch, scale, offset):
    """The fp32 filter works on float64 offsets to each simplex's center;
    its error bound must hold at any scale / offset (values stay bitwise
    the reference's)."""
    base = gen_sphere_torus_mix(40_000, seed=11).points
    X = base * scale + offset
    tri = delaunay(X[farthest_point_sampling(X, 150)])
    want = oracle.flood_values(X, tri.points, {k: tri.simplices_by_dim[k] for k in range(3)}, 10,
                               top_dim=2)
    for algo in (0, 1):
        algo_switch(algo)
        got = flood_sq_values(X, tri, 10, True, 2)
        for k in range(3):
            assert np.array_equal(got[k], want[k]), (algo, k)


def test_near_ties_lattice_cloud(algo_switch):
    """A jittered lattice: many candidates at nearly equal distances from
    sample points, where the fp32 minimum and the float64 minimum can pick
    different points; the refine must still return the float64 value."""
    g = np.stack(np.meshgrid(np.arange(30.0), np.arange(30.0), np.arange(30.0)), -1).reshape(-1, 3)
    X = g + np.random.default_rng(2).normal(scale=1e-7, size=g.shape)
    tri = delaunay(X[farthest_point_sampling(X, 120)])
    want = oracle.flood_values(X, tri.points, tri.simplices_by_dim, 6)
    for algo in (0, 1):
        algo_switch(algo)
        got = flood_sq_values(X, tri, 6, True)
        for k in range(4):
            assert np.array_equal(got[k], want[k]), (algo, k)


def test_concurrent_host_threads_share_the_device():
    """Four host threads value different complexes on one device at once
    (host-memory calls on the library stream and device-memory calls on
    their own torch streams): the grid-parameter slot the search kernels
    read is serialised per device, so every result stays bit-exact."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    from paper_2509_22432_b200.batch import DeviceComplex, flood_sq_device

    names = ["rand3d_m4", "torus10k_m20", "rand3d_m30", "dup3d_m5", "circle_m64", "rand2d_m6"]

    def host_call(name):
        z = G.load("flood", name)
        tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
        subset = str(z["landmark_mode"]) == "subset"
        sq = flood_sq_values(z["points"], tri, int(z["grid_resolution"]), subset)
        return all(np.array_equal(np.sqrt(sq[k]), want) for k, want in G.values_by_dim(z).items())

    def device_call(name):
        z = G.load("flood", name)
        tri = C.triangulation(z["tri_points"], G.simplices_by_dim(z))
        dev = torch.device("cuda:0")
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            X = torch.from_numpy(np.ascontiguousarray(z["points"])).to(dev)
            dc = DeviceComplex(tri, dev)
            got = [v.cpu().numpy() for v in flood_sq_device(X, dc, int(z["grid_resolution"]))]
        s.synchronize()
        return all(np.array_equal(np.sqrt(got[k]), want) for k, want in G.values_by_dim(z).items())

    with ThreadPoolExecutor(4) as pool:
        futs = [pool.submit(host_call if i % 2 else device_call, names[i % len(names)])
                for i in range(16)]
        assert all(f.result() for f in futs)


@pytest.mark.parametrize("dim,world", [(3, 2), (3, 5), (3, 8), (2, 4)])
def test_spatial_shards_equal_single_gpu(dim, world):
    """fph_flood_subset over spatially compact shards (the bench's multi-GPU
    partition), computed rank after rank on one GPU, reassembled and
    completed: equal to the single-call values."""
    import torch

    from paper_2509_22432_b200.parallel import (complete, simplex_centers, spatial_partition,
                                                subset_interior)

    if dim == 3:
        X = gen_sphere_torus_mix(150_000, seed=4).points
    else:
        X = np.random.default_rng(4).random((120_000, 2))
    top = dim
    tri = delaunay(X[farthest_point_sampling(X, 400)])
    want = flood_sq_values(X, tri, 10, True, top)
    dev = torch.device("cuda:0")
    Xd = torch.from_numpy(X).to(dev)
    lm = torch.from_numpy(np.ascontiguousarray(tri.points)).to(dev)
    by_dim = {k: torch.from_numpy(np.ascontiguousarray(tri.simplices_by_dim[k], dtype=np.int32)).to(dev)
              for k in range(top + 1)}
    fac = {k: torch.from_numpy(np.ascontiguousarray(tri.facet_links[k], dtype=np.int32)).to(dev)
           for k in range(1, top + 1)}
    parts = {k: [torch.from_numpy(p).to(dev) for p in
                 spatial_partition(simplex_centers(tri.points, tri.simplices_by_dim[k]), None, world)]
             for k in range(1, top + 1)}
    interior = {k: torch.full((by_dim[k].shape[0],), float("nan"), dtype=torch.float64, device=dev)
                for k in range(1, top + 1)}
    for r in range(world):
        share = subset_interior(Xd, lm, by_dim, top, 10, True, {k: parts[k][r] for k in range(1, top + 1)})
        for k in range(1, top + 1):
            interior[k][parts[k][r]] = share[k]
    got = complete(interior, fac, by_dim[0].shape[0], top, True)
    for k in range(top + 1):
        assert np.array_equal(got[k].cpu().numpy(), want[k]), k
