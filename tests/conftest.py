"""Shared fixtures.  `-m gpu` tests need a B200 and librafem_b200.so; the
rest run on CPU (oracle vs golden vectors, ABI exports, host logic)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def golden_meshes():
    with open(os.path.join(GOLDEN, "meshes.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def reference():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference package not present on this machine")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import rafem  # noqa: F401
    import rafem.fem, rafem.mesh, rafem.solver, rafem.sparse  # noqa: E401,F401
    return rafem
