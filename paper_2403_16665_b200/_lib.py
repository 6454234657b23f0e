"""ctypes binding of the C ABI in include/asx.h (libasx.so, built in-tree).

There is no CPU fallback: if the library is missing the import of any
compute entry point raises, and on a machine without a GPU every compute
call fails with ``AsxCudaError``.
"""

from __future__ import annotations

import ctypes
import os

from .core import UnsupportedSizeError

LIB_PATH = os.environ.get("ASX_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libasx.so")

ASX_OK = 0
ASX_ERR_INVALID = 2
ASX_ERR_INCOMPATIBLE = 3
ASX_ERR_UNSUPPORTED = 4
ASX_ERR_CUDA = 10
ASX_ERR_OOM = 11

ASX_C64 = 0
ASX_C128 = 1

ASX_AUTO, ASX_DIRECT, ASX_FFT, ASX_CHIRP = 0, 1, 2, 3
METHODS = {"auto": ASX_AUTO, "direct": ASX_DIRECT, "naive": ASX_DIRECT, "fft": ASX_FFT, "chirp": ASX_CHIRP}
METHOD_NAMES = {ASX_AUTO: "auto", ASX_DIRECT: "direct", ASX_FFT: "fft", ASX_CHIRP: "chirp"}


class AsxCudaError(RuntimeError):
    """CUDA failure inside libasx (no device, launch failure, out of memory)."""


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("m", ctypes.c_int64),
        ("a_num", ctypes.c_int64),
        ("a_den", ctypes.c_int64),
        ("m_ref", ctypes.c_int64),
        ("depth", ctypes.c_int32),
        ("leaf", ctypes.c_int32),
        ("method", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("real_input", ctypes.c_int32),
        ("fft_size", ctypes.c_int32),
        ("predicted_mults", ctypes.c_int64),
        ("predicted_adds", ctypes.c_int64),
        ("workspace_bytes", ctypes.c_int64),
        ("kernels_per_execute", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("batch_group", ctypes.c_int64),
    ]


# name -> (restype, argtypes); must match include/asx.h (tests/test_abi.py checks it)
_I64 = ctypes.c_int64
_VP = ctypes.c_void_p
SIGNATURES = {
    "asx_version": (ctypes.c_int, []),
    "asx_plan_create": (
        ctypes.c_int,
        [ctypes.POINTER(_VP), _I64, _I64, _I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int],
    ),
    "asx_execute": (ctypes.c_int, [_VP, _VP, _I64, _VP, _I64, _I64, _VP]),
    "asx_execute_host": (ctypes.c_int, [_VP, _VP, _I64, _VP, _I64, _I64, _I64]),
    "asx_plan_query": (ctypes.c_int, [_VP, ctypes.POINTER(PlanInfo)]),
    "asx_plan_destroy": (ctypes.c_int, [_VP]),
    "asx_dft_matrix": (ctypes.c_int, [_I64, _I64, _I64, _I64, ctypes.c_int, _VP, _VP]),
    "asx_combine": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _I64, ctypes.c_int, _VP]),
    "asx_block_sum": (ctypes.c_int, [_VP, _VP, _I64, _I64, ctypes.c_int, _VP]),
    "asx_last_launch": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)] * 4),
    "asx_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "asx_last_error": (ctypes.c_char_p, []),
}

_LIB = None


def lib() -> ctypes.CDLL:
    """Load libasx.so once; raise loudly if it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`)."
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def last_error() -> str:
    msg = lib().asx_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "libasx") -> None:
    """Map an asx_status to the reference's exception types (ref/core.py:17-31)."""
    if status == ASX_OK:
        return
    msg = f"{what}: {last_error() or lib().asx_strerror(status).decode()}"
    if status == ASX_ERR_UNSUPPORTED:
        raise UnsupportedSizeError(msg)
    if status in (ASX_ERR_INVALID, ASX_ERR_INCOMPATIBLE):
        raise ValueError(msg)
    raise AsxCudaError(msg)
