"""Run the REFERENCE's own test suite with the INTEGRATION.md ctypes stub
patched into it (the two call-site edits INTEGRATION.md shows), on a GPU box.

Inputs (git-ignored, they travel to the GPU box with the snapshot):
  baseline/_ref/floodph        the reference installed with
                               pip install --no-index --no-build-isolation --no-deps
                               --target baseline/_ref <copy of /root/reference/pkg>
  baseline/_ref/floodph_tests  the reference's tests/ directory (copied beside it)

The patched copy is built under /tmp; nothing under the repo is modified.

  python tools/integration/run_reference_suite.py [pytest args...]
"""

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
STUB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "floodph_b200_stub.py")
LIB = os.path.join(ROOT, "paper_2509_22432_b200", "_lib", "libfloodph_b200.so")

FPS_EDIT = '''

# --- B200 integration (INTEGRATION.md): farthest point sampling on the GPU
from . import _b200 as _b200_mod  # noqa: E402


def farthest_point_sampling(cloud, k: int, start: int = 0) -> np.ndarray:  # noqa: F811
    return _b200_mod.farthest_point_sampling(as_points(cloud), int(k), int(start))
'''

VALUES_OLD = '''        if backend == "masked-batch":
            msq_by_dim = _grid_values_masked(pts, tri, config, timings)
        else:
            msq_by_dim = _grid_values_kdtree(pts, tri, config, subset_mode, timings)'''
VALUES_NEW = '''        from . import _b200  # B200 integration (INTEGRATION.md)

        t0 = time.perf_counter()
        msq_by_dim = _b200.grid_values(pts, tri, config, subset_mode)
        timings[STAGE_FILTRATION] += time.perf_counter() - t0'''


def main():
    work = "/tmp/floodph_b200_suite"
    shutil.rmtree(work, ignore_errors=True)
    shutil.copytree(os.path.join(REF, "floodph"), os.path.join(work, "floodph"))
    shutil.copytree(os.path.join(REF, "floodph_tests"), os.path.join(work, "tests"))
    pkg = os.path.join(work, "floodph")
    shutil.copy(STUB, os.path.join(pkg, "_b200.py"))
    with open(os.path.join(pkg, "geometry.py"), "a") as fh:
        fh.write(FPS_EDIT)
    path = os.path.join(pkg, "filtration.py")
    src = open(path).read()
    if VALUES_OLD not in src:
        raise SystemExit("reference filtration.py differs from the expected call site")
    open(path, "w").write(src.replace(VALUES_OLD, VALUES_NEW))
    env = dict(os.environ, PYTHONPATH=work, FLOODPH_B200_LIB=LIB)
    cmd = [sys.executable, "-m", "pytest", os.path.join(work, "tests"), "-q", "-p", "no:cacheprovider",
           *sys.argv[1:]]
    print(" ".join(cmd), flush=True)
    # the patched package must be the one imported, and the GPU library loaded
    check = subprocess.run([sys.executable, "-c",
                            "import floodph, floodph._b200 as b, floodph.geometry as g;"
                            "print(floodph.__file__, b._lib, g.farthest_point_sampling.__module__)"],
                           env=env, cwd=work, capture_output=True, text=True)
    print(check.stdout.strip(), check.stderr.strip()[-500:], flush=True)
    sys.exit(subprocess.run(cmd, env=env, cwd=work).returncode)


if __name__ == "__main__":
    main()
