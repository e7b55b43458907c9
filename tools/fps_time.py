"""Time farthest point sampling on BASELINE configs (CUDA events, best of 5).

    python tools/fps_time.py        # on a GPU box
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_22432_b200.datagen import gen_sphere_torus_mix, gen_uniform_box  # noqa: E402
from paper_2509_22432_b200.geometry import farthest_point_sampling, farthest_point_sampling_batched  # noqa: E402


def timed(fn):
    best = 1e30
    out = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, out


def main():
    X = torch.from_numpy(gen_sphere_torus_mix(1_000_000, seed=0).points).cuda()
    ms, idx = timed(lambda: farthest_point_sampling(X, 2000, 0))
    print(f"sphere_torus_1m k=2000: {ms:.2f} ms  checksum {int(np.asarray(idx.cpu() if torch.is_tensor(idx) else idx).sum())}")
    B = torch.from_numpy(np.stack([gen_uniform_box(100_000, seed=s).points for s in range(64)])).cuda()
    ms, idx = timed(lambda: farthest_point_sampling_batched(B, 1000, 0))
    print(f"batched 64 x 100k k=1000: {ms:.2f} ms")
    if "--tiled" in sys.argv:
        T = torch.from_numpy(gen_uniform_box(10_000_000, seed=0).points).cuda()
        ms, idx = timed(lambda: farthest_point_sampling(T, 5000, 0))
        print(f"box_10m k=5000 (tiled): {ms:.2f} ms")


if __name__ == "__main__":
    main()
