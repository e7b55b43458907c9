"""FPS time against the number of landmarks k on a bench workload's cloud
(CUDA events, best of 3): the slope is the per-iteration cost.

  python tools/fps_k.py --config box_10m
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    from paper_2509_22432_b200.geometry import farthest_point_sampling

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="box_10m")
    ap.add_argument("--ks", type=int, nargs="+", default=[2, 100, 1000, 2000, 5000])
    args = ap.parse_args()
    kind, n, nl, m, md = bench.CONFIGS[args.config]
    T = torch.from_numpy(bench._cloud(kind, n)).cuda()

    def timed(k):
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            farthest_point_sampling(T, k, 0)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    for k in args.ks:
        print(args.config, k, round(timed(k), 3))


if __name__ == "__main__":
    main()
