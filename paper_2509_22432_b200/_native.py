"""ctypes binding of libfloodph_b200.so (C ABI: include/floodph_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises.  Buffers are numpy arrays (host
calls) or torch CUDA tensors (device calls); torch is used only for device
memory and streams.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB_PATH
from .errors import IntegrityError

FPH_OK, FPH_EARG, FPH_ECUDA, FPH_ENOMEM, FPH_EINTEGRITY = 0, 1, 2, 3, 4
FPH_MEM_HOST, FPH_MEM_DEVICE = 0, 1

_d = ctypes.POINTER(ctypes.c_double)
_i32 = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); kept in sync with include/floodph_b200.h
SIGNATURES = {
    "fph_abi_version": (ctypes.c_int, []),
    "fph_last_error": (ctypes.c_char_p, []),
    "fph_device_count": (ctypes.c_int, []),
    "fph_farthest_point_sampling": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32,
                                                   ctypes.c_int64, ctypes.c_int64, _vp,
                                                   ctypes.c_int32, _vp]),
    "fph_farthest_point_sampling_batched": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64,
                                                           ctypes.c_int32, ctypes.c_int64,
                                                           ctypes.c_int64, _vp, ctypes.c_int32,
                                                           _vp]),
    "fph_flood_interior": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp,
                                          ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32,
                                          _vp]),
    "fph_flood_samples": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int64,
                                         _vp, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int32,
                                         ctypes.c_int32, _vp, ctypes.c_int32, _vp]),
    "fph_flood_filtration": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp,
                                            ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp,
                                            ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32,
                                            _vp]),
    "fph_flood_shard": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int64,
                                       ctypes.c_int32, _vp, _vp, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32, _vp]),
    "fph_flood_subset": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int64,
                                        ctypes.c_int32, _vp, _vp, _vp, _vp, ctypes.c_int32,
                                        ctypes.c_int32, _vp, ctypes.c_int32, _vp]),
    "fph_flood_complete": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp,
                                          _vp]),
    "fph_candidate_mask": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int64,
                                          _vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp,
                                          ctypes.c_int64]),
    "fph_persistence_pairs": (ctypes.c_int, [ctypes.c_int32, _vp, _vp, _vp, ctypes.c_int32, _vp,
                                             _vp]),
    "fph_set_tuning": (ctypes.c_int, [ctypes.c_double, ctypes.c_double]),
    "fph_set_search": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "fph_set_exact_pairs": (ctypes.c_int, [ctypes.c_double]),
    "fph_set_exact_candidates": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64]),
    "fph_set_profiling": (ctypes.c_int, [ctypes.c_int32]),
    "fph_flood_stats": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "fph_debug_simplex_cycles": (ctypes.c_int, [ctypes.c_int32, _vp, ctypes.c_int64, _vp]),
    "fph_fp32_peak_tflops": (ctypes.c_double, []),
    "fph_tmem_min_rate": (ctypes.c_double, []),
    "fph_tilemin_rate": (ctypes.c_double, []),
    "fph_launch_count": (ctypes.c_int64, [ctypes.c_int32]),
}

_lib = None


def load(path: str | None = None):
    """Load (once) and return the library handle; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("FPH_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA library not built ({path}); run `python -m paper_2509_22432_b200._build` "
            "or __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:  # an older build loaded through FPH_LIB for an A/B run
            if path == LIB_PATH:
                raise RuntimeError(f"{path} does not export {name}")
            continue
        fn.restype = res
        fn.argtypes = args
    if lib.fph_abi_version() != 1:
        raise RuntimeError("libfloodph_b200 ABI mismatch")
    _lib = lib
    return lib


def require_gpu():
    lib = load()
    if lib.fph_device_count() < 1:
        raise RuntimeError("paper_2509_22432_b200 needs a CUDA device (no CPU fallback)")
    return lib


def check(rc: int) -> None:
    if rc == FPH_OK:
        return
    msg = (load().fph_last_error() or b"").decode(errors="replace")
    if rc == FPH_EARG:
        raise ValueError(msg)
    if rc == FPH_EINTEGRITY:
        raise IntegrityError(msg)
    raise RuntimeError(f"libfloodph_b200 error {rc}: {msg}")


def ptr(a) -> int:
    """Address of a numpy array or torch tensor buffer."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def ptr_array(items, ctype):
    arr = (ctypes.c_void_p * len(items))()
    for i, it in enumerate(items):
        arr[i] = ptr(it) if it is not None else None
    return arr
