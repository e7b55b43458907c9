"""Kernel launches of ONE rank's share (fph_flood_subset over a spatial
part of a bench workload at world size W), bracketed by cudaProfilerStart /
Stop so that ncu sees only that call:

  ncu --profile-from-start off --metrics gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/shard_launches.csv \
      python tools/shard_launches.py --config sphere_torus_1m --world 8 --rank 0

Without ncu it prints the call's event-timed duration (median of 5, L2
flushed), which is the figure to set the serialised kernel list against.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2509_22432_b200 import _native
    from paper_2509_22432_b200.parallel import simplex_centers, spatial_partition, subset_interior

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sphere_torus_1m")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    args = ap.parse_args()
    _native.require_gpu()
    w = bench.prepare(args.config, 0)
    Xd, dc = w["items"][0]
    tri = w["tri"]
    by_dim = {0: torch.arange(dc.counts_full[0], dtype=torch.int32, device=dc.dev), **dc.simp}
    parts = {k: torch.from_numpy(spatial_partition(simplex_centers(tri.points, tri.simplices_by_dim[k]),
                                                   None, args.world)[args.rank]).to(dc.dev)
             for k in range(1, dc.top + 1)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dc.dev)

    def call():
        return subset_interior(Xd, dc.lm, by_dim, dc.top, w["m"], True, parts)

    times = []
    for _ in range(6):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    call()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(json.dumps({"config": args.config, "world": args.world, "rank": args.rank,
                      "rows": {k: int(v.shape[0]) for k, v in parts.items()},
                      "call_ms_median": float(np.median(times[1:]))}))


if __name__ == "__main__":
    main()
