"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/khb200.h declares, and the product path refuses to run without a GPU
(no CPU fallback)."""

import os
import re

import numpy as np
import pytest

from paper_2008_01996_b200 import _native

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "khb200.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kh_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES), "ctypes table and header disagree"


def test_status_strings_and_version():
    lib = _native.load()
    assert lib.kh_version() >= 1
    for code in range(6):
        assert lib.kh_status_string(code)


def test_invalid_arguments_map_to_exceptions():
    import ctypes

    from paper_2008_01996_b200.errors import DimensionMismatch, UsageError

    lib = _native.load()
    with pytest.raises(UsageError):
        _native.check(lib.kh_analyze(3, None, None, 0, None))
    indptr = np.array([0, 1, 2], np.int64)
    indices = np.array([0, 5], np.int64)  # out of range
    raw = ctypes.c_void_p()
    with pytest.raises(DimensionMismatch):
        _native.check(lib.kh_analyze(2, indptr.ctypes.data, indices.ctypes.data, 0, ctypes.byref(raw)))
    with pytest.raises(DimensionMismatch):
        _native.check(lib.kh_dgemm(4, 4, 4, 1.0, None, 2, None, 4, 0.0, None, 4, None))


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from conftest import load_golden
    from paper_2008_01996_b200 import solvers
    from paper_2008_01996_b200.errors import DeviceError

    system, _ = load_golden("lshape0")
    with pytest.raises(DeviceError):
        solvers.solve_fd(system)
    with pytest.raises(DeviceError):
        solvers.residual(system, system.rhs)
