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
