"""The north star's tensor-core question, measured.

As a GEMM the flooding kernel's distance pass is [a, |a|^2] . [-2b, 1]
(K = 4 of tf32's K = 8): every (sample point, candidate) product lands in TMEM
and must be read out (tcgen05.ld) and min-reduced.  This prints the measured
rate of that epilogue ALONE next to the FFMA2 tile-min loop the kernel runs:
if the epilogue by itself is slower than the whole FFMA2 pass, no tcgen05
variant can win, whatever its MMA throughput.

  python tools/tensor_core_decision.py > profiles/r02/tensor_core_decision.json
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2509_22432_b200 import _native

    lib = _native.require_gpu()
    tmem = lib.fph_tmem_min_rate()
    tile = lib.fph_tilemin_rate()
    ffma2 = lib.fph_fp32_peak_tflops()
    out = {
        "tmem_ld_min_elements_per_s": tmem,
        "ffma2_tilemin_pairs_per_s": tile,
        "ffma2_peak_tflops": ffma2,
        "ffma2_tilemin_pairs_per_s_at_peak": ffma2 * 1e12 / 8.0,  # 3 FFMA2 + 1 FMNMX3 per 2 pairs
        "epilogue_over_ffma2": tmem / tile if tile else None,
        "verdict": ("tcgen05 variant cannot win: reading the products out of TMEM alone is slower "
                    "than the complete FFMA2 pass" if tile and tmem < tile else
                    "epilogue is not the limiter: an MMA variant needs a full implementation to decide"),
        "precision_note": "tf32 keeps 10 mantissa bits: the certified error bound of the filter "
                          "grows 2^13 = 8192x against fp32, widening the float64 refine set",
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
