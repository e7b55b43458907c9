"""Per-simplex cost anatomy of the bounded search (debug capture of
fph_flood_interior: cycles of each simplex in the phase kernels A, B, C, F,
claim to publish; blocks searched / pruned, candidates staged, team size),
plus the heaviest simplices -- the ones that bound a shard's time at high
GPU counts -- against the average load per resident warp.

  python tools/simplex_costs.py [--config sphere_torus_1m] [--top 10]
                                [--world W --rank r]   (one rank's spatial share)

(record fields: cycles A, B, C, F; blocks searched; candidate count;
candidates staged; team size)
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2509_22432_b200 import _native

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sphere_torus_1m")
    ap.add_argument("--top", type=int, default=10)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    args = ap.parse_args()
    from paper_2509_22432_b200.parallel import simplex_centers, spatial_partition
    lib = _native.require_gpu()
    w = bench.prepare(args.config, 0)
    X, tri = w["X"], w["tri"]
    lms = np.ascontiguousarray(tri.points)
    out = {"config": args.config, "world": args.world, "rank": args.rank}
    clock_ghz = 1.965
    for k in range(1, w["max_dim"] + 1):
        rows = tri.simplices_by_dim[k]
        if args.world > 1:
            rows = rows[spatial_partition(simplex_centers(lms, rows), None, args.world)[args.rank]]
        s4 = np.full((rows.shape[0], 4), -1, dtype=np.int32)
        s4[:, : k + 1] = rows
        sq = np.empty(rows.shape[0])
        lib.fph_debug_simplex_cycles(1, None, 0, None)
        _native.check(lib.fph_flood_interior(_native.ptr(X), X.shape[0], X.shape[1], _native.ptr(lms),
                                             lms.shape[0], _native.ptr(s4), rows.shape[0], k, w["m"], 1,
                                             _native.ptr(sq), _native.FPH_MEM_HOST, None))
        n = np.zeros(1, dtype=np.int64)
        lib.fph_debug_simplex_cycles(0, None, 0, n.ctypes.data)
        buf = np.empty(int(n[0]), dtype=np.int64)
        lib.fph_debug_simplex_cycles(0, buf.ctypes.data, buf.size, n.ctypes.data)
        d = buf[2: 2 + 16 * int(buf[1])].reshape(-1, 16)
        tot = d[:, :4].sum(1).astype(float)
        staged = d[:, 6].astype(float)
        order = np.argsort(-tot)
        q = np.quantile(tot, [0.5, 0.9, 0.99, 0.999, 1.0])
        top1 = order[: max(1, len(order) // 100)]
        out[f"dim{k}"] = {
            "n": int(len(rows)),
            "warp_cycles_total": float(tot.sum()),
            "quantiles_warp_cycles_p50_p90_p99_p999_max": [float(v) for v in q],
            "max_simplex_us_single_warp": float(q[-1] / clock_ghz / 1e3),
            "mean_load_per_warp_us": float(tot.sum() / 2368 / clock_ghz / 1e3),
            "max_phase_us": [float(d[:, i].max() / clock_ghz / 1e3) for i in range(4)],
            "top1pct_share": float(tot[top1].sum() / tot.sum()),
            "phase_share": [float(d[:, i].sum() / tot.sum()) for i in range(4)],
            "team_simplices": int((d[:, 7] > 1).sum()),
            # simplices valued by one exact pass in phase A (no B / C work)
            "exact_pass_simplices": int(((d[:, 1] == 0) & (d[:, 2] == 0)).sum()),
            "exact_pass_share_of_A": float(d[(d[:, 1] == 0) & (d[:, 2] == 0), 0].sum() /
                                           max(d[:, 0].sum(), 1)),
            "exact_pass_share_of_all": float(d[(d[:, 1] == 0) & (d[:, 2] == 0), :4].sum() /
                                             max(tot.sum(), 1)),
            "cost_vs_cand_loglog_slope": float(np.polyfit(np.log(np.maximum(d[:, 5], 1)),
                                                          np.log(np.maximum(tot, 1)), 1)[0]),
            "cost_per_cand_by_cand_decile": [
                float(np.median(tot[(d[:, 5] >= lo) & (d[:, 5] <= hi)] /
                                np.maximum(d[(d[:, 5] >= lo) & (d[:, 5] <= hi), 5], 1)))
                for lo, hi in zip(np.quantile(d[:, 5], np.linspace(0, 0.9, 10)),
                                  np.quantile(d[:, 5], np.linspace(0.1, 1.0, 10)))],
            "heaviest_cand_rank_pct": [float((d[:, 5] < d[i, 5]).mean() * 100) for i in order[:10]],
            "heaviest": [{"row": int(i), "warp_cycles": float(tot[i]),
                          "phases": [int(v) for v in d[i, :4]], "blocks": int(d[i, 4]),
                          "cand": int(d[i, 5]), "staged": int(staged[i]), "team": int(d[i, 7])}
                         for i in order[: args.top]],
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
