"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/floodph_b200.h declares."""

import os
import re

import pytest

from paper_2509_22432_b200 import _build, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "floodph_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(fph_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_loads():
    path = _build.build()
    assert os.path.exists(path)
    lib = _native.load()
    assert lib.fph_abi_version() == 1


def test_exports_every_declared_symbol():
    lib = _native.load()
    declared = _declared()
    assert len(declared) >= 8
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.SIGNATURES)


def test_sass_targets_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly_on_cpu_box():
    lib = _native.load()
    if lib.fph_device_count() > 0:
        pytest.skip("GPU present")
    import numpy as np

    from paper_2509_22432_b200 import farthest_point_sampling

    with pytest.raises(RuntimeError):
        farthest_point_sampling(np.zeros((4, 2)), 2)


def test_argument_errors_match_reference_without_gpu():
    import numpy as np

    from paper_2509_22432_b200 import farthest_point_sampling

    with pytest.raises(ValueError):
        farthest_point_sampling(np.zeros((4, 2)), 0)
    with pytest.raises(ValueError):
        farthest_point_sampling(np.zeros((4, 2)), 5)
    with pytest.raises(ValueError):
        farthest_point_sampling(np.zeros((4, 2)), 2, start=4)
