"""The C-ABI library loads, exports every symbol include/asx.h declares, and
validates arguments on the host (no compute, no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_2403_16665_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "asx.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    decls = re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(asx_\w+)\s*\(([^;]*?)\)\s*;", text, flags=re.M | re.S)
    return {name: ([] if args.strip() in ("", "void") else args.split(",")) for name, args in decls}


def test_library_present_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "build libasx.so first (__graft_entry__.build())"
    assert _lib.lib().asx_version() == 2


def test_every_header_symbol_exported_with_matching_arity():
    declared = _declared()
    assert len(declared) >= 11
    handle = _lib.lib()
    for name, args in declared.items():
        assert hasattr(handle, name), name
        assert name in _lib.SIGNATURES, name
        assert len(_lib.SIGNATURES[name][1]) == len(args), name


def test_strerror_and_codes():
    L = _lib.lib()
    assert b"incompatible" in L.asx_strerror(3)
    assert b"unsupported" in L.asx_strerror(4)
    assert L.asx_strerror(0) == b"ok"


def _create(n, a, d, m=0, dtype=1, method=0):
    h = ctypes.c_void_p()
    rc = _lib.lib().asx_plan_create(ctypes.byref(h), n, a, d, m, dtype, 0, method, 0)
    if rc == 0:
        _lib.lib().asx_plan_destroy(h)
    return rc


def test_host_side_validation_needs_no_gpu():
    assert _create(0, 1, 2) == _lib.ASX_ERR_INVALID
    assert _create(8, 0, 2) == _lib.ASX_ERR_INVALID
    assert _create(8, 1, 2, dtype=7) == _lib.ASX_ERR_INVALID
    # alpha_b = 37/100 at N=256 has no integral alpha*N: IncompatibleAlphaError w/o explicit m
    assert _create(256, 37, 100) == _lib.ASX_ERR_INCOMPATIBLE
    assert "incompatible" in _lib.last_error()
    # reference plan() size rules (fastpath.py:97-101): N=12 is not a power of two
    assert _create(12, 1, 1, method=_lib.ASX_FFT) == _lib.ASX_ERR_UNSUPPORTED
    # alpha_ref = 3/2 -> alpha_b = 2/3: no power-of-two recursion
    assert _create(8, 2, 3, method=_lib.ASX_FFT) == _lib.ASX_ERR_UNSUPPORTED


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc = _create(1024, 1, 4, m=1024)
    assert rc == _lib.ASX_ERR_CUDA
    assert _lib.last_error()
    with pytest.raises(_lib.AsxCudaError):
        _lib.check(rc)


def test_null_and_negative_arguments():
    L = _lib.lib()
    assert L.asx_execute(None, None, 0, None, 0, 1, None) == _lib.ASX_ERR_INVALID
    assert L.asx_plan_query(None, None) == _lib.ASX_ERR_INVALID
    assert L.asx_plan_destroy(None) == 0
    assert L.asx_combine(None, None, None, None, -1, 2, 1, None) == _lib.ASX_ERR_INVALID
    assert L.asx_block_sum(None, None, 0, 4, 1, None) == 0
