"""Test configuration: `gpu` marker, import paths, shared fixtures.

``-m "not gpu"`` runs here (no GPU): the oracle against the reference-made
golden fixtures, the host-side logic, and the C-ABI symbol table.
``-m gpu`` runs on the B200: parity of the CUDA path against the oracle and
the golden fixtures.
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libocpgpu.so")
    config.addinivalue_line("markers", "slow: long-running case")


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def native_gpu():
    """Loads the library and checks a device is visible; fails loudly otherwise."""
    from paper_2411_00546_b200 import _native
    from paper_2411_00546_b200._build import build
    build()
    return _native.load()
