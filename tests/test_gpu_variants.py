"""GPU: the big-cloud build of the search kernels (slot 2: 4 CTAs per SM,
64 registers, 128-candidate tiles; taken for clouds of >= 64 MiB) passes
the same parity suite when every call is forced onto it
(FPH_BIG_MIN_BYTES=0).  Run in a fresh process: the threshold is read once
per process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_big_cloud_kernels_pass_the_parity_suite():
    env = dict(os.environ, FPH_BIG_MIN_BYTES="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-q",
                        "-x", "-k", "not fps", "-p", "no:cacheprovider"],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
    assert " passed" in r.stdout


def test_sorted_fps_kernel_passes_the_fps_suite():
    """The Morton-sorted resident FPS kernel (taken by clouds of >= 262144
    points) forced onto every cloud (FPH_FPS_SORTED_MIN=0): every FPS parity
    test -- goldens, oracle, ties, each points-per-thread instantiation --
    gives the reference's indices."""
    env = dict(os.environ, FPH_FPS_SORTED_MIN="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-q",
                        "-x", "-k", "fps", "-p", "no:cacheprovider"],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
    assert " passed" in r.stdout
