"""Per-rank cost table of the sharded flood filtration, measured on ONE GPU.

For a bench workload and world sizes W, times every rank's share
(fph_flood_shard, rank r of W: grid build + interior terms of rows r, r + W,
...) one after another, the facet completion, and the single-GPU call, with
CUDA events and an L2 flush before each.  The step at W GPUs is bounded by
the slowest rank, so the predicted strong-scaling efficiency is

    eff(W) = T_1 / (W * (max_r T_r + T_complete + T_gather)),

T_gather the all-gather of the interior values (one float64 per simplex),
taken as GATHER_US (NVLink latency-bound at these sizes).

  python tools/shard_costs.py --config box_10m --worlds 2 4 8
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GATHER_US = 40.0  # assumed: one NCCL all-gather of <= 1 MB across 8 GPUs over NVSwitch


def main():
    import torch

    import bench
    from paper_2509_22432_b200 import _native
    from paper_2509_22432_b200.batch import flood_sq_device
    from paper_2509_22432_b200.parallel import (complete, shard_interior, simplex_centers,
                                                spatial_partition, subset_interior)

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sphere_torus_1m")
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--strategies", nargs="+", default=["interleaved", "spatial", "spatial_cand"])
    args = ap.parse_args()
    _native.require_gpu()
    w = bench.prepare(args.config, 0)
    Xd, dc = w["items"][0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dc.dev)
    vert_ids = torch.arange(dc.counts_full[0], dtype=torch.int32, device=dc.dev)
    by_dim = {0: vert_ids, **dc.simp}

    def timed(fn):
        best = []
        for _ in range(args.reps + 1):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1))
        return float(np.median(best[1:])), out

    lib = _native.require_gpu()
    stats = np.zeros(24)

    grid_ms = []

    def interiors_ms(fn, keep=None):
        """(call ms, fork-to-join ms of the interior kernels inside it)"""
        lib.fph_set_profiling(1)
        lib.fph_flood_stats(stats.ctypes.data, 1)
        t, out = timed(fn)
        lib.fph_flood_stats(stats.ctypes.data, 1)
        lib.fph_set_profiling(0)
        if keep is not None:
            keep.append(out)
        grid_ms.append(stats[23] / (args.reps + 1))
        return t, stats[6] / (args.reps + 1)

    t1, _ = timed(lambda: flood_sq_device(Xd, dc, w["m"]))
    # fixed cost of a share: a world so large each dimension keeps one simplex
    fixed, fixed_int = interiors_ms(
        lambda: shard_interior(Xd, dc.lm, by_dim, dc.top, w["m"], True, 0, 1 << 30))
    one, one_int = interiors_ms(lambda: flood_sq_device(Xd, dc, w["m"]))
    tri = w["tri"]
    cand = {}
    if "spatial_cand" in args.strategies:  # Lemma-4.2 candidate counts as the cost model
        for k in range(1, dc.top + 1):
            cells = np.ascontiguousarray(tri.simplices_by_dim[k], dtype=np.int32)
            offs = np.zeros(cells.shape[0] + 1, dtype=np.int64)
            X = np.ascontiguousarray(w["X"])
            lms = np.ascontiguousarray(tri.points)
            _native.check(lib.fph_candidate_mask(_native.ptr(X), X.shape[0], X.shape[1],
                                                 _native.ptr(lms), lms.shape[0], _native.ptr(cells),
                                                 cells.shape[0], k, _native.ptr(offs), None, 0))
            cand[k] = np.diff(offs).astype(np.float64)
    centers = {k: simplex_centers(tri.points, tri.simplices_by_dim[k]) for k in range(1, dc.top + 1)}
    rows = []
    for strategy in args.strategies:
        for W in args.worlds:
            per, per_int = [], []
            interior = {k: torch.empty(dc.counts_full[k], dtype=torch.float64, device=dc.dev)
                        for k in range(1, dc.top + 1)}
            if strategy != "interleaved":
                parts = {k: [torch.from_numpy(p).to(dc.dev) for p in
                             spatial_partition(centers[k], cand.get(k) if strategy == "spatial_cand"
                                               else None, W)]
                         for k in range(1, dc.top + 1)}
            for r in range(W):
                keep = []
                if strategy == "interleaved":
                    fn = lambda: shard_interior(Xd, dc.lm, by_dim, dc.top, w["m"], True, r, W)  # noqa: E731
                else:
                    fn = lambda: subset_interior(Xd, dc.lm, by_dim, dc.top, w["m"], True,  # noqa: E731
                                                 {k: parts[k][r] for k in parts})
                t, ti = interiors_ms(fn, keep)
                share = keep[0]
                per.append(t)
                per_int.append(ti)
                for k in range(1, dc.top + 1):
                    if strategy == "interleaved":
                        interior[k][r::W] = share[k]
                    else:
                        interior[k][parts[k][r]] = share[k]
            tc, vals = timed(lambda: complete(interior, dc.facets, dc.counts_full[0], dc.top, True))
            ref = flood_sq_device(Xd, dc, w["m"])
            same = all(torch.equal(vals[k], ref[k]) for k in range(dc.top + 1))
            step = max(per) + tc + GATHER_US / 1e3
            rows.append({"strategy": strategy, "world": W, "rank_ms": per, "rank_interiors_ms": per_int,
                         "max_rank_ms": max(per), "mean_rank_ms": float(np.mean(per)),
                         "imbalance": max(per) / float(np.mean(per)), "complete_ms": tc,
                         "predicted_step_ms": step, "predicted_efficiency": t1 / (W * step),
                         "reassembled_equals_single": same})
    print(json.dumps({"config": args.config, "simplices": dc.n_simplices, "single_gpu_ms": t1,
                      "single_call_interiors_ms": one_int, "fixed_share_ms": fixed,
                      "fixed_share_interiors_ms": fixed_int,
                      "grid_build_ms": grid_ms[0] if grid_ms else None,
                      "gather_us_assumed": GATHER_US, "worlds": rows}))


if __name__ == "__main__":
    main()
