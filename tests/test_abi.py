"""C-ABI surface: the library loads and exports every symbol include/ocp_gpu.h declares.

No compute call is made (the build container has no GPU); creating a context
without a device must fail cleanly with OCP_ERR_NO_DEVICE, not crash.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from paper_2411_00546_b200 import _native
from paper_2411_00546_b200._build import build

HEADER = os.path.join(REPO, "include", "ocp_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ocp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _native.load()


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ("ocp_ctx_create", "ocp_raspen_residual", "ocp_raspen_jvp", "ocp_mgs",
                 "ocp_vec_nrm2", "ocp_local_residual", "ocp_local_direction"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared_symbols()) == set(_native.SIGNATURES)


def test_no_device_is_a_clean_error(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    f = np.zeros(16)
    ctx = ctypes.c_void_p()
    rc = lib.ocp_ctx_create(4, 1, 1, 0, 1e-3, 1e-2, 1, 0.0, _native.ptr(f), _native.ptr(f),
                            ctypes.byref(ctx))
    assert rc == _native.OCP_ERR_NO_DEVICE
    assert "device" in _native.last_error(None)


def test_argument_errors_mirror_decompose(lib):
    f = np.zeros(9)
    ctx = ctypes.c_void_p()
    rc = lib.ocp_ctx_create(3, 4, 1, 0, 1e-3, 1e-2, 1, 0.0, _native.ptr(f), _native.ptr(f),
                            ctypes.byref(ctx))
    assert rc == _native.OCP_ERR_ARG
    assert "nonempty" in _native.last_error(None)
    f = np.zeros(64)
    rc = lib.ocp_ctx_create(8, 2, 1, 5, 1e-3, 1e-2, 1, 0.0, _native.ptr(f), _native.ptr(f),
                            ctypes.byref(ctx))
    assert rc == _native.OCP_ERR_ARG
    assert "row direction" in _native.last_error(None)
