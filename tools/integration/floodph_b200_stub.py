# floodph/_b200.py  (new file in the reference package)
import ctypes, os
import numpy as np

_lib = ctypes.CDLL(os.environ.get("FLOODPH_B200_LIB", "libfloodph_b200.so"))
_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib.fph_farthest_point_sampling.argtypes = [_vp, _i64, _i32, _i64, _i64, _vp, _i32, _vp]
_lib.fph_flood_filtration.argtypes = [_vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp, _vp,
                                      _i32, _i32, _vp, _i32, _vp]
_lib.fph_last_error.restype = ctypes.c_char_p
HOST = 0

def _check(rc):
    if rc == 1:
        raise ValueError(_lib.fph_last_error().decode())
    if rc:
        raise RuntimeError(_lib.fph_last_error().decode())

def farthest_point_sampling(pts, k, start=0):
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    out = np.empty(k, dtype=np.int64)
    _check(_lib.fph_farthest_point_sampling(pts.ctypes.data, pts.shape[0], pts.shape[1],
                                            k, start, out.ctypes.data, HOST, None))
    return out

def grid_values(pts, tri, config, subset_mode):
    """Drop-in for filtration._grid_values_masked / _grid_values_kdtree."""
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    lms = np.ascontiguousarray(tri.points, dtype=np.float64)
    top = tri.dim
    counts = np.array([tri.simplices_by_dim[k].shape[0] for k in range(top + 1)], np.int64)
    keep = []
    def table(arrays):
        t = (ctypes.c_void_p * (top + 1))()
        for k, a in enumerate(arrays):
            if a is not None:
                keep.append(a); t[k] = a.ctypes.data
        return t
    simp = [None] + [np.ascontiguousarray(tri.simplices_by_dim[k], np.int32) for k in range(1, top + 1)]
    fac = [None] + [np.ascontiguousarray(tri.facet_links[k], np.int32) for k in range(1, top + 1)]
    outs = [np.empty(max(int(c), 1)) for c in counts]
    _check(_lib.fph_flood_filtration(
        pts.ctypes.data, pts.shape[0], pts.shape[1], lms.ctypes.data, lms.shape[0], top,
        counts.ctypes.data, table(simp), table(fac), config.grid_resolution,
        1 if subset_mode else 0, table(outs), HOST, None))
    return {k: outs[k][: counts[k]] for k in range(top + 1)}
