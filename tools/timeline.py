"""Timeline of one flooding step (profiling aid): every simplex's phase
intervals from the global timer (debug capture), turned into the number of
busy warps over time, against the resident capacity -- where the step's idle
warp-time sits (start-up, between phases, tail).

  python tools/timeline.py [--config sphere_torus_1m] [--bins 60]
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2509_22432_b200 import _native
    from paper_2509_22432_b200.batch import flood_sq_device

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sphere_torus_1m")
    ap.add_argument("--bins", type=int, default=60)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    args = ap.parse_args()
    lib = _native.require_gpu()
    w = bench.prepare(args.config, 0)
    Xd, dc = w["items"][0]
    call = lambda: flood_sq_device(Xd, dc, w["m"])  # noqa: E731
    if args.world > 1:  # one rank's spatial share (fph_flood_subset)
        from paper_2509_22432_b200.parallel import simplex_centers, spatial_partition, subset_interior

        tri = w["tri"]
        by_dim = {0: torch.arange(dc.counts_full[0], dtype=torch.int32, device=dc.dev), **dc.simp}
        parts = {k: torch.from_numpy(spatial_partition(simplex_centers(tri.points, tri.simplices_by_dim[k]),
                                                       None, args.world)[args.rank]).to(dc.dev)
                 for k in range(1, dc.top + 1)}
        call = lambda: subset_interior(Xd, dc.lm, by_dim, dc.top, w["m"], True, parts)  # noqa: E731
    for _ in range(3):
        call()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dc.dev)
    flush.zero_()
    torch.cuda.synchronize()
    lib.fph_debug_simplex_cycles(1, None, 0, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    n = np.zeros(1, dtype=np.int64)
    lib.fph_debug_simplex_cycles(0, None, 0, n.ctypes.data)
    buf = np.empty(int(n[0]), dtype=np.int64)
    lib.fph_debug_simplex_cycles(0, buf.ctypes.data, buf.size, n.ctypes.data)
    recs, pos = [], 0
    while pos < buf.size:
        k, cnt = int(buf[pos]), int(buf[pos + 1])
        d = buf[pos + 2: pos + 2 + 16 * cnt].reshape(-1, 16)
        recs.append((k, d))
        pos += 2 + 16 * cnt
    t0 = min(int(d[:, 8:16:2][d[:, 8:16:2] > 0].min()) for _, d in recs)
    t1 = max(int(d[:, 9:16:2].max()) for _, d in recs)
    span_us = (t1 - t0) / 1e3
    edges = np.linspace(0, span_us, args.bins + 1)
    busy = np.zeros(args.bins)
    per_phase = {}
    for k, d in recs:
        team = np.maximum(d[:, 7], 1)
        for ph in range(4):
            s, e = d[:, 8 + 2 * ph], d[:, 9 + 2 * ph]
            m = (s > 0) & (e > s)
            if not m.any():
                continue
            s_us, e_us = (s[m] - t0) / 1e3, (e[m] - t0) / 1e3
            per_phase[f"dim{k}_{'ABCF'[ph]}"] = [float(s_us.min()), float(e_us.max()), int(m.sum())]
            for a, b, t in zip(s_us, e_us, team[m]):
                lo = np.searchsorted(edges, a, side="right") - 1
                hi = np.searchsorted(edges, b, side="left")
                for i in range(max(lo, 0), min(hi, args.bins)):
                    ov = min(b, edges[i + 1]) - max(a, edges[i])
                    if ov > 0:
                        busy[i] += t * ov / (edges[i + 1] - edges[i])
    # resident warps: 148 SMs x 8 warps x CTAs per SM (2; 4 for the big-cloud
    # build, clouds of >= 64 MiB, fph_flood.cuh kBigSlot)
    big = Xd.shape[0] * Xd.shape[1] * 8 >= (64 << 20)
    capacity = 148.0 * 8 * (4 if big else 2)
    out = {"config": args.config, "world": args.world, "rank": args.rank,
           "step_ms_events": e0.elapsed_time(e1),
           "first_claim_to_last_publish_us": span_us,
           "busy_warps_by_bin": [round(float(b), 1) for b in busy],
           "bin_us": float(edges[1] - edges[0]), "capacity_warps": capacity,
           "mean_utilisation": float(busy.mean() / capacity),
           "phase_windows_us": per_phase}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
