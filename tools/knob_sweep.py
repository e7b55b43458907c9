"""Sweep the bounded search's knobs (representative sample size, CTA-team
threshold) on a bench workload: single-GPU step and, for a world size W,
the slowest rank's share (interleaved shards), CUDA events, L2 flushed.

  python tools/knob_sweep.py --config box_10m --world 8 --reps 512 2048 --team 0 -100 -50
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
    from paper_2509_22432_b200.parallel import shard_interior

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="box_10m")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--reps", type=int, nargs="+", default=[512])
    ap.add_argument("--team", type=int, nargs="+", default=[0])
    ap.add_argument("--exact-pairs", type=float, nargs="+", default=[65536.0])
    ap.add_argument("--exact-cand2", type=int, nargs="+", default=[1000])
    ap.add_argument("--exact-cand1", type=int, nargs="+", default=[0])
    args = ap.parse_args()
    lib = _native.require_gpu()
    w = bench.prepare(args.config, 0)
    Xd, dc = w["items"][0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dc.dev)
    by_dim = {0: torch.arange(dc.counts_full[0], dtype=torch.int32, device=dc.dev), **dc.simp}

    def timed(fn, reps=3):
        out = []
        for _ in range(reps + 1):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return float(np.median(out[1:]))

    rows = []
    import itertools

    for reps, team, ep, ec, ec1 in itertools.product(args.reps, args.team, args.exact_pairs,
                                                     args.exact_cand2, args.exact_cand1):
        if True:
            _native.check(lib.fph_set_search(1, reps, team))
            _native.check(lib.fph_set_exact_pairs(ep))
            _native.check(lib.fph_set_exact_candidates(2, ec))
            _native.check(lib.fph_set_exact_candidates(1, ec1))
            t1 = timed(lambda: flood_sq_device(Xd, dc, w["m"]))
            W = args.world
            per = [timed(lambda: shard_interior(Xd, dc.lm, by_dim, dc.top, w["m"], True, r, W), 1)
                   for r in range(W)] if W > 1 else [t1]
            rows.append({"reps": reps, "team": team, "exact_pairs": ep, "exact_cand2": ec,
                         "exact_cand1": ec1,
                         "single_ms": t1, "max_rank_ms": max(per),
                         "mean_rank_ms": float(np.mean(per)),
                         "predicted_efficiency": t1 / (W * (max(per) + 0.05))})
            print(json.dumps(rows[-1]), flush=True)
    _native.check(lib.fph_set_search(1, 0, 0))
    _native.check(lib.fph_set_exact_pairs(-1))
    _native.check(lib.fph_set_exact_candidates(2, 1000))
    _native.check(lib.fph_set_exact_candidates(1, 0))


if __name__ == "__main__":
    main()
