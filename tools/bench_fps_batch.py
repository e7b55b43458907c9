"""configs[3] FPS stage: a batch of ModelNet-sized synthetic clouds (100k
points, 1k landmarks each) through the batched FPS kernel; prints clouds/s
and ms per cloud (CUDA events, device-resident input)."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2509_22432_b200 import farthest_point_sampling, farthest_point_sampling_batched
    from paper_2509_22432_b200.datagen import gen_sphere_torus_mix

    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    n, k = 100_000, 1000
    clouds = np.stack([gen_sphere_torus_mix(n, seed=s).points for s in range(batch)])
    X = torch.from_numpy(clouds).cuda()
    farthest_point_sampling_batched(X[:2], 8)
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("batched", lambda: farthest_point_sampling_batched(X, k)),
                     ("one_by_one", lambda: [farthest_point_sampling(X[b], k) for b in range(batch)])):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[name] = {"ms": ms, "clouds_per_s": batch / (ms / 1e3), "ms_per_cloud": ms / batch}
    a = farthest_point_sampling_batched(X, k).cpu().numpy()
    b = np.stack([farthest_point_sampling(X[i], k).cpu().numpy() for i in range(batch)])
    res["identical"] = bool((a == b).all())
    print(json.dumps({"workload": "configs[3] FPS stage", "batch": batch, "points": n,
                      "landmarks": k, **res}))


if __name__ == "__main__":
    main()
