"""GPU: batches of clouds (BASELINE configs[3] path, batch.flood_cloud_batch):
one batched FPS launch, host Delaunay on a thread pool, per-cloud device
flood values -- every cloud's landmarks and values equal the oracle's."""

import numpy as np
import pytest

import oracle
from paper_2509_22432_b200.batch import flood_cloud_batch
from paper_2509_22432_b200.datagen import gen_modelnet_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("max_dim", [None, 2])
def test_cloud_batch_matches_oracle(max_dim):
    clouds = gen_modelnet_batch(5, 30_000, seed=7)
    rep = flood_cloud_batch(clouds, 300, m=8, max_dim=max_dim, workers=3)
    assert [r.cloud for r in rep.results] == list(range(5))
    for r in rep.results:
        X = clouds[r.cloud]
        np.testing.assert_array_equal(r.landmark_indices, oracle.fps(X, 300, 0))
        tri = r.triangulation
        top = tri.dim if max_dim is None else max_dim
        want = oracle.flood_values(X, tri.points, {k: tri.simplices_by_dim[k] for k in range(top + 1)},
                                   8, top_dim=top)
        assert sorted(r.sq_values) == list(range(top + 1))
        for k in range(top + 1):
            assert np.array_equal(r.sq_values[k], want[k]), (r.cloud, k)
    assert rep.timings["fps_s"] > 0 and rep.timings["flood_s"] > 0


def test_two_grid_slots_in_flight_equal_one_at_a_time():
    """Clouds dealt to two streams (the library's two constant grid slots,
    two calls in flight) -- eagerly and inside a CUDA graph -- give exactly
    the values of one call at a time."""
    import torch

    from paper_2509_22432_b200 import farthest_point_sampling
    from paper_2509_22432_b200.batch import DeviceComplex, flood_sq_device, flood_sq_device_many
    from paper_2509_22432_b200.delaunay import delaunay

    dev = torch.device("cuda:0")
    clouds = gen_modelnet_batch(6, 40_000, seed=11)
    items = []
    for X in clouds:
        Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
        idx = farthest_point_sampling(Xd, 400, 0).cpu().numpy()
        items.append((Xd, DeviceComplex(delaunay(X[idx]), dev)))
    want = []
    for Xd, dc in items:
        want.append([v.clone() for v in flood_sq_device(Xd, dc, 10)])
        torch.cuda.synchronize()
    for out in items:
        for v in out[1].out:
            v.fill_(float("nan"))
    got = flood_sq_device_many(items, 10)
    torch.cuda.synchronize()
    for g, w in zip(got, want):
        assert all(torch.equal(a, b) for a, b in zip(g, w))
    s = torch.cuda.Stream(device=dev)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=s, capture_error_mode="thread_local"):
        flood_sq_device_many(items, 10, True, s.cuda_stream)
    for _, dc in items:
        for v in dc.out:
            v.fill_(float("nan"))
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for (_, dc), w in zip(items, want):
        assert all(torch.equal(dc.out[k][: dc.counts_full[k]], w[k]) for k in range(dc.top + 1))


def test_second_grid_slot_kernels_bit_exact():
    """FPH_GRID_SLOTS=2 (both compiled copies of the search kernels in use,
    two calls' searches in flight): the same values as one call at a time.
    Run in a fresh process, since the slot count is read once per process."""
    import os
    import subprocess
    import sys

    script = r'''
import numpy as np, torch
from paper_2509_22432_b200 import farthest_point_sampling
from paper_2509_22432_b200.batch import DeviceComplex, flood_sq_device, flood_sq_device_many
from paper_2509_22432_b200.datagen import gen_modelnet_batch
from paper_2509_22432_b200.delaunay import delaunay
dev = torch.device("cuda:0")
items = []
for X in gen_modelnet_batch(5, 30_000, seed=3):
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
    idx = farthest_point_sampling(Xd, 300, 0).cpu().numpy()
    items.append((Xd, DeviceComplex(delaunay(X[idx]), dev)))
want = []
for Xd, dc in items:
    want.append([v.clone() for v in flood_sq_device(Xd, dc, 9)])
    torch.cuda.synchronize()
for _ in range(2):
    got = flood_sq_device_many(items, 9)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for g, w in zip(got, want) for a, b in zip(g, w))
print("ok")
'''
    env = dict(os.environ, FPH_GRID_SLOTS="2")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", script], env=env, cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
