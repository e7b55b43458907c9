"""Sweep the grid's cell occupancy (points per cell the cell edge is sized
for, fph_set_tuning) on bench workloads: single-call step, CUDA events,
L2 flushed, median of 5.

  python tools/occupancy_sweep.py --configs sphere_torus_1m box_10m --occ 1 1.5 2 3 4
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
    ap.add_argument("--configs", nargs="+", default=["sphere_torus_1m"])
    ap.add_argument("--occ", type=float, nargs="+", default=[1.0, 1.5, 2.0, 3.0, 4.0])
    args = ap.parse_args()
    lib = _native.require_gpu()
    for cfg in args.configs:
        w = bench.prepare(cfg, 0)
        Xd, dc = w["items"][0]
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dc.dev)
        ref = None
        for occ in args.occ:
            _native.check(lib.fph_set_tuning(occ, 0.0))
            times = []
            for _ in range(6):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                out = flood_sq_device(Xd, dc, w["m"])
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            vals = [v.clone() for v in out]
            same = ref is None or all(torch.equal(a, b) for a, b in zip(vals, ref))
            ref = ref or vals
            print(json.dumps({"config": cfg, "occupancy": occ, "ms": float(np.median(times[1:])),
                              "values_equal": same}))
        _native.check(lib.fph_set_tuning(0.0, 0.0))


if __name__ == "__main__":
    main()
