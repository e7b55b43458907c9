"""Build libfloodph_b200.so in-tree with nvcc for sm_100a.

The shared library lands in paper_2509_22432_b200/_lib/ (git-ignored; it
travels to the GPU box with the repo snapshot).  Each source compiles to its
own object in parallel (no device code crosses files), then one link.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libfloodph_b200.so")
SOURCES = ["fph_api.cu", "fph_flood.cu", "fph_search.cu", "fph_fps.cu", "fph_grid.cu",
           "fph_diag.cu", "fph_mask.cu", "fph_persistence.cpp"]
HEADERS = ["fph_common.cuh", "fph_dev.cuh", "fph_flood.cuh", "fph_grid.cuh"]
# compiled again per extra grid slot (-DFPH_GRID_SLOT=g, g = 1 .. GRID_SLOTS - 1)
SLOTTED = ["fph_search.cu"]
GRID_SLOTS = 3
# slot 2: the build for clouds beyond L2 (fph_flood.cuh kBigSlot)
SLOT_DEFINES = {2: ["-DFPH_SEARCH_MINB=4", "-DFPH_WT=128", "-DFPH_VALS_CAP=256"]}

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the CUDA library")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "floodph_b200.h"))
    return any(os.path.getmtime(d) > built for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines=()) -> str:
    """Compile the library if any source is newer than it; return its path.

    `out` / `defines` build an experimental variant (tuning A/B runs)."""
    target = out or LIB_PATH
    if not force and out is None and not _stale():
        return LIB_PATH
    os.makedirs(os.path.dirname(target), exist_ok=True)
    objdir = target + ".objs"
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    defs = [f"-D{d}" for d in defines]

    def compile_one(unit):
        src, extra = unit
        obj = os.path.join(objdir, src + "".join(e.replace("=", "").replace("-D", "_") for e in extra) + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *defs, *extra, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        return obj

    # the search kernels once per constant grid slot (fph_flood.cuh kGridSlots)
    units = [(src, []) for src in SOURCES]
    units += [(src, [f"-DFPH_GRID_SLOT={g}", *SLOT_DEFINES.get(g, [])]) for src in SLOTTED
              for g in range(1, GRID_SLOTS)]
    with ThreadPoolExecutor(max_workers=len(units)) as pool:
        objs = list(pool.map(compile_one, units))
    tmp = target + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    shutil.rmtree(objdir, ignore_errors=True)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
