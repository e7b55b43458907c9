"""Time the flooding pass of BASELINE configs[1] under different tunings.

Prints one line per setting: ms per pass (CUDA events around the C-ABI call,
device buffers), pair / staging counters.  Values are asserted identical to
the first setting's (all settings are exact).
"""

import itertools
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import DeviceComplex, prepare, step_single
    from paper_2509_22432_b200 import _native

    cfg = sys.argv[1] if len(sys.argv) > 1 else "sphere_torus_1m"
    settings = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [
        [1, 1024, 32768, 8.0], [0, 0, 0, 8.0]]
    lib = _native.require_gpu()
    w = prepare(cfg, 0)
    dc = DeviceComplex(w, 0)
    stream = torch.cuda.current_stream().cuda_stream
    ref = None
    stats = np.zeros(24)
    for st in settings:
        algo, reps, team, occ = st[:4]
        exact = st[4] if len(st) > 4 else -1
        ecand = st[5] if len(st) > 5 else [0, 0, 0, 0]
        for kk in range(4):
            lib.fph_set_exact_candidates(kk, int(ecand[kk]))
        _native.check(lib.fph_set_search(algo, reps, team))
        lib.fph_set_exact_pairs(float(exact))
        lib.fph_set_tuning(occ, 0.0)
        step_single(lib, _native, w, dc, stream)
        torch.cuda.synchronize()
        lib.fph_set_profiling(1)
        lib.fph_flood_stats(stats.ctypes.data, 1)
        times = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step_single(lib, _native, w, dc, stream)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        lib.fph_flood_stats(stats.ctypes.data, 1)
        lib.fph_set_profiling(0)
        vals = [t.cpu().numpy().copy() for t in dc.out]
        same = None
        if ref is None:
            ref = vals
        else:
            same = all(np.array_equal(a, b) for a, b in zip(ref, vals))
        s = stats / 3
        print(json.dumps({"algo": algo, "reps": reps, "team": team, "occ": occ, "exact": exact, "ecand": ecand,
                          "ms": round(min(times), 3), "pass_ms": round(s[6], 3), "pairs": s[0],
                          "staged": s[1], "refined": s[3], "blocks": s[7], "pruned_blocks": s[8],
                          "team_simplices": s[9], "st_A": s[16], "st_Csample": s[17],
                          "st_Cfull": s[18], "cyc_A": s[19], "cyc_B": s[20], "cyc_C": s[21],
                          "cyc_F": s[22], "searches": s[15], "cyc_prologue": s[2], "same": same}),
              flush=True)


if __name__ == "__main__":
    main()
