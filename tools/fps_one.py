"""One FPS call on a bench workload's cloud (for ncu captures of the FPS
kernels): python tools/fps_one.py --config box_10m --k 1000"""
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
    ap.add_argument("--k", type=int, default=1000)
    args = ap.parse_args()
    kind, n, nl, m, md = bench.CONFIGS[args.config]
    T = torch.from_numpy(bench._cloud(kind, n)).cuda()
    farthest_point_sampling(T, args.k, 0)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
