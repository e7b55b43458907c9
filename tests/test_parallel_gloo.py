"""Multi-rank host logic of the sharded flood filtration, world size 2, gloo
on CPU.  Interior values come from the CPU oracle (test infrastructure);
the code under test is the sharding, the all-gather back into row order and
the facet completion identity used by bench.py / parallel.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_22432_b200.parallel import flood_sq_values_sharded, gather_interleaved, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_rows_partition():
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            parts = [shard_rows(n, world, r) for r in range(world)]
            allrows = np.sort(np.concatenate(parts))
            np.testing.assert_array_equal(allrows, np.arange(n))
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)


def _worker(rank, world, port, payload, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        interior = payload["interior"]
        facets = payload["facets"]
        values = {0: np.zeros(payload["n0"])}
        for k in sorted(interior):
            full = interior[k]
            mine = torch.from_numpy(full[shard_rows(full.shape[0], world, rank)])
            got = gather_interleaved(mine, full.shape[0], world, dist).numpy()
            assert np.array_equal(got, full)
            values[k] = np.maximum(got, values[k - 1][facets[k]].max(axis=1))
        q.put((rank, {k: v.tolist() for k, v in values.items()}))
    finally:
        dist.destroy_process_group()


def test_sharded_gather_and_completion_world2():
    import oracle
    from tests import _complex as C
    from tests import _golden as G

    z = G.load("flood", "rand3d_m4")
    by_dim = G.simplices_by_dim(z)
    tri = C.triangulation(z["tri_points"], by_dim)
    m = int(z["grid_resolution"])
    # full values are valid "interior" inputs: completion is idempotent on
    # a monotone complex (max(f(s), f(facets)) == f(s))
    full = oracle.flood_values(z["points"], z["tri_points"], by_dim, m)
    interior = {k: full[k] for k in range(1, 4)}
    payload = {"interior": interior, "facets": tri.facet_links, "n0": by_dim[0].shape[0]}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, payload, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        for k in range(1, 4):
            assert np.array_equal(np.asarray(results[r][k]), full[k])
            assert np.array_equal(np.sqrt(np.asarray(results[r][k])), z[f"values_{k}"])


def _cpu_complete(interior, facets, n0, top, subset):
    out = {0: torch.zeros(n0, dtype=torch.float64)}
    for k in range(1, top + 1):
        lower = out[k - 1][torch.from_numpy(np.asarray(facets[k]))]
        out[k] = torch.maximum(interior[k], lower.max(dim=1).values)
    return out


def _worker_e2e(rank, world, port, payload, q):
    """flood_sq_values_sharded end to end on gloo: the rank's interior share
    (host stand-in for fph_flood_shard: rows rank, rank + world, ...), the
    all-gather, and the completion."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        interior = payload["interior"]
        by_dim = {k: torch.from_numpy(v) for k, v in payload["by_dim"].items()}

        def interior_fn(r, w):
            assert (r, w) == (rank, world)
            return {k: torch.from_numpy(interior[k][r::w].copy()) for k in interior}

        vals = flood_sq_values_sharded(None, None, by_dim, payload["facets"], 3,
                                       payload["m"], dist, interior_fn=interior_fn,
                                       complete_fn=_cpu_complete)
        q.put((rank, {k: v.numpy().tolist() for k, v in vals.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_flood_sq_values_sharded_end_to_end(world):
    from tests import _complex as C
    from tests import _golden as G

    z = G.load("flood", "dup3d_m5")
    by_dim = G.simplices_by_dim(z)
    tri = C.triangulation(z["tri_points"], by_dim)
    vals = G.values_by_dim(z)
    # interior terms: the reference's own squared values (completion is
    # idempotent on a monotone complex, so they are valid interior inputs)
    interior = {k: vals[k] ** 2 for k in range(1, 4)}
    payload = {"interior": interior, "facets": tri.facet_links, "m": int(z["grid_resolution"]),
               "by_dim": {k: np.asarray(v) for k, v in by_dim.items()}}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_e2e, args=(r, world, port, payload, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert np.array_equal(np.asarray(results[r][0]), np.zeros(by_dim[0].shape[0]))
        for k in range(1, 4):
            assert np.array_equal(np.sqrt(np.asarray(results[r][k])), vals[k]), (r, k)


def _worker_partitioned(rank, world, port, payload, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_22432_b200.parallel import gather_partitioned, spatial_partition

        parts = [torch.from_numpy(p) for p in spatial_partition(payload["centers"], None, world)]
        full = payload["values"]
        mine = torch.from_numpy(full[parts[rank].numpy()])
        got = gather_partitioned(mine, parts, full.shape[0], world, dist).numpy()
        q.put((rank, bool(np.array_equal(got, full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_spatial_partition_gather(world):
    """Spatially compact shards (Morton cuts of the simplex centers, the same
    on every rank) gathered back into row order over gloo."""
    from paper_2509_22432_b200.parallel import simplex_centers, spatial_partition
    from tests import _golden as G

    z = G.load("flood", "torus10k_m20")
    rows = z["simplices_2"]
    centers = simplex_centers(z["tri_points"], rows)
    parts = spatial_partition(centers, None, world)
    assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(rows.shape[0]))
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    payload = {"centers": centers, "values": z["values_2"] ** 2}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_partitioned, args=(r, world, port, payload, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(results.values())
