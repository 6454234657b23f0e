"""Drop-in α-DFT / α-FFT API, executed by libasx.so on a B200.

Same names, argument meaning and error behaviour as the reference's L2 layer
(/root/reference/pkg/src/alpha_spectra/, cited ``ref/<file>:<line>``):

=====================  ==========================================  ========================
this module            reference                                   device path
=====================  ==========================================  ========================
``dft_matrix``         ref/oracle.py:26-34                         k_dft_matrix
``naive_forward``      ref/oracle.py:50-67                         k_direct (method direct)
``plan`` / ``Plan``    ref/fastpath.py:63-110                      asx_plan_create
``transform_samples``  ref/fastpath.py:162-181                     k_afft / k_chirp
``alpha_fft``          ref/fastpath.py:184-194                     k_afft / k_chirp
``combine``            ref/fastpath.py:130-151                     k_combine
``leaf_block_sum``     ref/fastpath.py:154-159                     k_block_sum
``predicted_mults``    ref/fastpath.py:113-121                     closed form
``predicted_adds``     ref/fastpath.py:124-127                     closed form
``OpCounter``          ref/fastpath.py:45-60                       closed-form accounting
=====================  ==========================================  ========================

Additions: keyword ``m`` (explicit bin count), ``dtype``
(complex64 / complex128), ``method`` ('fft' = the α-FFT recursion, 'chirp',
'direct', 'auto'), batched 2-D inputs (rows = signals), and torch CUDA
tensors in/out without host copies.  Host (numpy) inputs go through the
C ABI's host-buffer entry point (copies inside).
"""

from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (
    DenseFactor,
    IncompatibleAlphaError,
    Signal,
    Spectrum,
    UnsupportedSizeError,
    validate_pair,
)


class LeafKind(enum.Enum):
    SINGLE_SAMPLE = "single_sample"  # alpha_ref >= 1 (ref/fastpath.py:41)
    BLOCK_SUM = "block_sum"  # alpha_ref < 1 (ref/fastpath.py:42)


@dataclass
class OpCounter:
    """Complex multiply/add tally (ref/fastpath.py:45-60).

    The GPU kernels do not count at run time; a transform adds the reference
    closed forms (ref/fastpath.py:113-127) per signal, which is what the
    reference's counter measures for its recursion.
    """

    complex_mults: int = 0
    complex_adds: int = 0

    def reset(self) -> None:
        self.complex_mults = 0
        self.complex_adds = 0


def _dtype_code(dtype) -> int:
    if dtype is None:
        return _lib.ASX_C128
    name = str(dtype).replace("torch.", "").replace("numpy.", "").replace("<class '", "").replace("'>", "")
    if name in ("complex64", "c64", "cfloat", "float32", "F"):
        return _lib.ASX_C64
    if name in ("complex128", "c128", "cdouble", "float64", "complex", "D"):
        return _lib.ASX_C128
    raise ValueError(f"unsupported dtype {dtype!r}: use complex64 or complex128")


_NP_COMPLEX = {_lib.ASX_C64: np.complex64, _lib.ASX_C128: np.complex128}
_NP_REAL = {_lib.ASX_C64: np.float32, _lib.ASX_C128: np.float64}


def _torch():
    import torch  # plumbing only: device memory and streams

    return torch


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


def _default_device() -> int:
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.AsxCudaError("no CUDA device is available (libasx has no CPU fallback)")
    return torch.cuda.current_device()


class Plan:
    """Validated (N, alpha, M) with device-resident tables (ref/fastpath.py:63-82).

    Immutable after construction; ``execute`` is safe from several streams.
    """

    def __init__(self, n, alpha: DenseFactor, m=None, dtype="complex128", method="fft",
                 real_input=False, device=None):
        if not isinstance(alpha, DenseFactor):
            raise TypeError("alpha must be a DenseFactor")
        if method not in _lib.METHODS:
            raise ValueError(f"unknown method {method!r}; one of {sorted(_lib.METHODS)}")
        self.alpha = alpha
        self._dtype = _dtype_code(dtype)
        self.real_input = bool(real_input)
        dev = _default_device() if device is None else int(device)
        handle = ctypes.c_void_p()
        # α_b = q/p: a_num = alpha.q, a_den = alpha.p
        status = _lib.lib().asx_plan_create(
            ctypes.byref(handle), int(n), alpha.q, alpha.p, 0 if m is None else int(m), self._dtype,
            int(self.real_input), _lib.METHODS[method], dev)
        if status == _lib.ASX_ERR_INCOMPATIBLE:
            raise IncompatibleAlphaError(int(n), alpha.p, alpha.q)
        _lib.check(status, "plan")
        self._handle = handle
        info = _lib.PlanInfo()
        _lib.check(_lib.lib().asx_plan_query(handle, ctypes.byref(info)), "plan_query")
        self.info = info
        self.n = int(info.n)
        self.m = int(info.m)
        self.m_ref = int(info.m_ref)
        self.depth = int(info.depth)
        self.leaf = {1: LeafKind.SINGLE_SAMPLE, 2: LeafKind.BLOCK_SUM}.get(info.leaf)
        self.method = _lib.METHOD_NAMES[info.method]
        self.fft_size = int(info.fft_size)
        self.device = dev
        self.predicted_mults = int(info.predicted_mults)
        self.predicted_adds = int(info.predicted_adds)
        self.workspace_bytes = int(info.workspace_bytes)
        self._twiddles = None
        self._lock = threading.Lock()

    # -- reference Plan surface ------------------------------------------
    @property
    def shape(self) -> tuple:
        return (self.m, self.n)

    @property
    def dtype(self):
        return _NP_COMPLEX[self._dtype]

    @property
    def twiddles(self) -> tuple:
        """Reference tables exp(-2πi l/(M_ref>>k)), l < (M_ref>>k)/2 (ref/fastpath.py:104-109).

        Generated on the device (k_dft_matrix with exact reduction), read-only.
        """
        if self._twiddles is None:
            tables = []
            for k in range(max(self.depth, 0)):
                size = self.m_ref >> k
                row = dft_matrix_rows(size, DenseFactor(1), 2, dtype="complex128", device=self.device)[1]
                t = np.array(row[: size // 2])
                t.setflags(write=False)
                tables.append(t)
            self._twiddles = tuple(tables)
        return self._twiddles

    # -- execution ---------------------------------------------------------
    def _in_dtype(self):
        return (_NP_REAL if self.real_input else _NP_COMPLEX)[self._dtype]

    def execute(self, x, out=None, stream=None):
        """Batched transform of a CUDA tensor x (..., N) -> (..., M); rows are signals.

        Leading dimensions are flattened into the batch and restored on the
        output (``out``, if given, must then be a (B, M) view with B their
        product)."""
        torch = _torch()
        if x.dim() == 0 or x.shape[-1] != self.n:
            raise ValueError(f"plan is for N={self.n}, got {tuple(x.shape)} samples")
        lead = tuple(x.shape[:-1])
        squeeze = x.dim() == 1
        xb = x.unsqueeze(0) if squeeze else (x.reshape(-1, self.n) if x.dim() > 2 else x)
        want = getattr(torch, np.dtype(self._in_dtype()).name)
        xb = xb.resolve_conj().resolve_neg()  # lazy conj/neg views would hand the kernel raw memory
        if xb.dtype != want:
            xb = xb.to(want)
        if xb.stride(-1) != 1:
            xb = xb.contiguous()
        if xb.device.type != "cuda":
            raise ValueError("execute() takes CUDA tensors; use execute_host() for host arrays")
        batch = xb.shape[0]
        cdt = getattr(torch, np.dtype(self.dtype).name)
        if out is None:
            out = torch.empty((batch, self.m), dtype=cdt, device=xb.device)
        else:
            out = out.view(batch, self.m) if out.dim() == 1 else out
            if out.dtype != cdt or out.stride(-1) != 1 or out.shape != (batch, self.m):
                raise ValueError("out must be a (B, M) tensor of the plan's complex dtype, unit inner stride")
        st = torch.cuda.current_stream(xb.device).cuda_stream if stream is None else int(stream)
        xs = xb.stride(0) if batch > 1 else self.n
        Xs = out.stride(0) if batch > 1 else self.m
        _lib.check(_lib.lib().asx_execute(self._handle, xb.data_ptr(), xs, out.data_ptr(), Xs, batch, st),
                   "execute")
        if squeeze:
            return out[0]
        return out.view(lead + (self.m,)) if len(lead) > 1 else out

    def execute_host(self, x, out=None, chunk: int = 0) -> np.ndarray:
        """Batched transform of a host array (B, N) or (N,); copies run inside the C ABI."""
        arr = np.asarray(x)
        if arr.ndim == 0 or arr.shape[-1] != self.n:
            raise ValueError(f"plan is for N={self.n}, got {arr.shape} samples")
        lead = arr.shape[:-1]
        squeeze = arr.ndim == 1
        arr = np.ascontiguousarray(arr.reshape(-1, self.n), dtype=self._in_dtype())
        batch = arr.shape[0]
        if out is None:
            out = np.empty((batch, self.m), dtype=self.dtype)
        elif out.dtype != self.dtype or not out.flags.c_contiguous or out.size != batch * self.m:
            raise ValueError("out must be a C-contiguous array of the plan's dtype and size B*M")
        _lib.check(_lib.lib().asx_execute_host(self._handle, arr.ctypes.data, self.n, out.ctypes.data,
                                               self.m, batch, int(chunk)), "execute_host")
        out = out.reshape(batch, self.m)
        if squeeze:
            return out[0]
        return out.reshape(lead + (self.m,)) if len(lead) > 1 else out

    def __call__(self, x, **kw):
        return self.execute(x, **kw) if _is_tensor(x) and x.device.type == "cuda" else self.execute_host(x, **kw)

    def close(self) -> None:
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            _lib.lib().asx_plan_destroy(h)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __repr__(self) -> str:
        return (f"Plan(n={self.n}, m={self.m}, alpha={self.alpha}, method={self.method}, "
                f"dtype={np.dtype(self.dtype).name}, fft_size={self.fft_size})")


def plan(n: int, alpha: DenseFactor, *, m=None, dtype="complex128", method="fft", real_input=False,
         device=None) -> Plan:
    """Validate (N, alpha) and build the device plan (ref/fastpath.py:85-110).

    Raises IncompatibleAlphaError when m is None and alpha*N is not an
    integer; UnsupportedSizeError when ``method`` cannot take the size (the
    'fft' method follows the reference's power-of-two rule, generalised to
    any integer density).
    """
    if m is None:
        validate_pair(n, alpha)
    return Plan(n, alpha, m=m, dtype=dtype, method=method, real_input=real_input, device=device)


_PLAN_CACHE: dict = {}
_PLAN_CACHE_LOCK = threading.Lock()


def _cached_plan(n, alpha, m, dtype, method, device, real_input=False) -> Plan:
    dev = _default_device() if device is None else int(device)
    key = (n, alpha.p, alpha.q, m, _dtype_code(dtype), method, dev, bool(real_input))
    with _PLAN_CACHE_LOCK:
        p = _PLAN_CACHE.get(key)
        if p is None:
            if len(_PLAN_CACHE) >= 64:
                _PLAN_CACHE.pop(next(iter(_PLAN_CACHE))).close()
            p = Plan(n, alpha, m=m, dtype=dtype, method=method, real_input=real_input, device=dev)
            _PLAN_CACHE[key] = p
        return p


def predicted_mults(p: Plan) -> int:
    """(alpha*N/2) * log2(min(N, alpha*N)) (ref/fastpath.py:113-121)."""
    return p.predicted_mults


def predicted_adds(p: Plan) -> int:
    """alpha*N per level plus block-sum leaf adds (ref/fastpath.py:124-127)."""
    return p.predicted_adds


def _count(counter: OpCounter | None, p: Plan, signals: int) -> None:
    if counter is not None and p.predicted_mults >= 0:
        counter.complex_mults += p.predicted_mults * signals
        counter.complex_adds += p.predicted_adds * signals


def transform_samples(x, p: Plan, counter: OpCounter | None = None):
    """Run the planned transform on bare samples (ref/fastpath.py:162-181).

    x: (N,) or (B, N) numpy array -> numpy bins; CUDA tensor -> CUDA tensor.
    """
    shape = tuple(x.shape)
    if not shape or shape[-1] != p.n:
        got = shape[0] if len(shape) == 1 else shape
        raise ValueError(f"plan is for N={p.n}, got {got} samples")
    out = p(x)
    _count(counter, p, int(np.prod(shape[:-1])) if len(shape) > 1 else 1)
    return out


def alpha_fft(signal: Signal, p: Plan, counter: OpCounter | None = None) -> Spectrum:
    """Fast density-alpha transform of ``signal`` (ref/fastpath.py:184-194)."""
    if len(signal) != p.n:
        raise ValueError(f"plan is for N={p.n}, signal has {len(signal)} samples")
    bins = transform_samples(signal.samples, p, counter)
    return Spectrum(np.asarray(bins, dtype=np.complex128), p.n, p.alpha, signal.duration,
                    m_bins=None if p.m == p.m_ref else p.m)


def naive_forward(signal: Signal, alpha: DenseFactor, *, m=None, dtype="complex128", device=None) -> Spectrum:
    """Direct α-DFT (ref/oracle.py:50-67) on the GPU: dense W[M, N] contraction."""
    n = len(signal)
    if m is None:
        m_eff = validate_pair(n, alpha).m
    else:
        m_eff = int(m)
    p = _cached_plan(n, alpha, m_eff if m is not None else None, dtype, "direct", device)
    bins = p.execute_host(signal.samples.astype(p.dtype) if p.dtype != np.complex128 else signal.samples)
    return Spectrum(np.asarray(bins, dtype=np.complex128), n, alpha, signal.duration,
                    m_bins=None if m is None else m_eff)


def dft_matrix_rows(n: int, alpha: DenseFactor, rows: int, *, dtype="complex128", device=None,
                    as_tensor=False):
    """First ``rows`` rows of the density-alpha matrix, built on the device."""
    torch = _torch()
    dev = _default_device() if device is None else int(device)
    code = _dtype_code(dtype)
    cdt = getattr(torch, np.dtype(_NP_COMPLEX[code]).name)
    W = torch.empty((rows, n), dtype=cdt, device=f"cuda:{dev}")
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().asx_dft_matrix(int(n), alpha.q, alpha.p, int(rows), code, W.data_ptr(), st),
               "dft_matrix")
    return W if as_tensor else W.cpu().numpy()


def dft_matrix(n: int, alpha: DenseFactor, *, m=None, dtype="complex128", device=None, as_tensor=False):
    """The (alpha*N) x N transform matrix, row m, column n = w^(m n) (ref/oracle.py:26-34).

    ``m`` selects a different row count (e.g. the first N rows, or any count
    for alpha values whose alpha*N is not integral).
    """
    rows = validate_pair(n, alpha).m if m is None else int(m)
    return dft_matrix_rows(n, alpha, rows, dtype=dtype, device=device, as_tensor=as_tensor)


def _as_device_pair(*arrays, dtype_code):
    torch = _torch()
    dev = _default_device()
    cdt = getattr(torch, np.dtype(_NP_COMPLEX[dtype_code]).name)
    outs = []
    for a in arrays:
        if _is_tensor(a):
            outs.append(a.to(device=f"cuda:{dev}", dtype=cdt).contiguous())
        else:
            outs.append(torch.from_numpy(np.ascontiguousarray(a, dtype=_NP_COMPLEX[dtype_code])).to(f"cuda:{dev}"))
    return outs, dev


def combine(y, z, twiddles, counter: OpCounter | None = None):
    """Butterfly merge [y + w z, y - w z] along the last axis (ref/fastpath.py:130-151)."""
    ys, zs, ts = tuple(np.shape(y)), tuple(np.shape(z)), tuple(np.shape(twiddles))
    if ys != zs:
        raise ValueError(f"half-spectra differ in shape: {ys} vs {zs}")
    if not ys or ys[-1] != ts[-1]:
        raise ValueError(
            f"twiddle table length {ts[-1] if ts else 0} does not match half-spectrum length {ys[-1] if ys else 0}")
    host = not _is_tensor(y)
    code = _lib.ASX_C128
    (yd, zd, td), dev = _as_device_pair(y, z, twiddles, dtype_code=code)
    half = ys[-1]
    rows = int(np.prod(ys[:-1])) if len(ys) > 1 else 1
    torch = _torch()
    out = torch.empty(ys[:-1] + (2 * half,), dtype=yd.dtype, device=yd.device)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().asx_combine(yd.data_ptr(), zd.data_ptr(), td.data_ptr(), out.data_ptr(), rows, half,
                                      code, st), "combine")
    if counter is not None:
        counter.complex_mults += rows * half
        counter.complex_adds += 2 * rows * half
    return out.cpu().numpy() if host else out


def leaf_block_sum(block, counter: OpCounter | None = None) -> complex:
    """Terminal 1 x (1/alpha) apply: the plain sum of a block (ref/fastpath.py:154-159)."""
    size = int(np.prod(np.shape(block)))
    if counter is not None and size > 0:
        counter.complex_adds += size - 1
    if size == 0:
        return 0j
    torch = _torch()
    (bd,), dev = _as_device_pair(np.reshape(block, -1) if not _is_tensor(block) else block.reshape(-1),
                                 dtype_code=_lib.ASX_C128)
    out = torch.empty((1,), dtype=bd.dtype, device=bd.device)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().asx_block_sum(bd.data_ptr(), out.data_ptr(), 1, size, _lib.ASX_C128, st),
               "block_sum")
    return complex(out.cpu().numpy()[0])


__all__ = [
    "LeafKind", "OpCounter", "Plan", "plan", "predicted_mults", "predicted_adds", "transform_samples",
    "alpha_fft", "naive_forward", "dft_matrix", "dft_matrix_rows", "combine", "leaf_block_sum",
    "UnsupportedSizeError",
]
