"""SURVEY.md §8(f) rows 1-2 on the GPU: the inverse α-DFT and the classical
comparators of the reference (ref/oracle.py:70-103, ref/baseline.py:24-97).

* ``naive_inverse``  x_n = (1/M) Σ_m X_m exp(+2πi m n / M), n < N
  (ref/oracle.py:70-87).  It is the forward transform of conj(X) with input
  length M, α = 1 and N outputs, conjugated and scaled — the same CUDA plans
  (method auto picks α-FFT / chirp / direct), no separate kernel.
* ``orthogonality_kernel`` (ref/oracle.py:90-103): entry (n-l) mod M of the
  inverse of an all-ones spectrum, computed by that inverse on the device.
* ``zero_pad`` / ``PaddedSignal`` (ref/baseline.py:24-64): host data layout only.
* ``standard_fft`` (ref/baseline.py:67-81): the α-FFT at density 1.
* ``aliased_reconstruct`` (ref/baseline.py:84-97): the BLOCK_SUM fold
  x'_n = Σ_k x_{n+kM}, summed by ``asx_block_sum`` on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DenseFactor, Signal, Spectrum, validate_pair
from .transforms import OpCounter, _cached_plan, _default_device, _torch, alpha_fft, plan


def _inverse_rows(X, n: int, device=None):
    """x[b, :n] = (1/M) conj(T(conj(X[b]))), T = α-DFT with input length M, α = 1."""
    torch = _torch()
    dev = _default_device() if device is None else int(device)
    Xt = X if (hasattr(X, "device") and getattr(X, "is_cuda", False)) else torch.from_numpy(
        np.array(X, dtype=np.complex128)).to(f"cuda:{dev}")
    Xt = Xt.to(torch.complex128)
    if Xt.dim() == 1:
        Xt = Xt.unsqueeze(0)
    m = Xt.shape[1]
    p = _cached_plan(m, DenseFactor(1), n, "complex128", "auto", dev)
    y = p.execute(torch.conj_physical(Xt).contiguous())
    return torch.conj_physical(y) / m


def naive_inverse(spectrum: Spectrum) -> Signal:
    """Literal inverse α-DFT (ref/oracle.py:70-87), on the GPU.

    For alpha >= 1 it recovers the signal; for alpha < 1 the alias-folded
    signal, extended periodically over n < N.
    """
    x = _inverse_rows(spectrum.bins, spectrum.origin_n)
    return Signal(x[0].cpu().numpy(), spectrum.duration)


def orthogonality_kernel(n_index: int, l_index: int, n: int, alpha: DenseFactor) -> complex:
    """(1/M) Σ_m exp(+2πi m (n-l)/M) (ref/oracle.py:90-103): 1 on the alias comb, ~0 off it."""
    _, m = validate_pair(n, alpha)
    delta = (n_index - l_index) % m
    if delta == 0:
        return 1.0 + 0j  # the comb point is exactly 1 (the reference divides an exact sum of ones)
    comb = _inverse_rows(np.ones(m, dtype=np.complex128), m)
    return complex(comb[0, delta].item())


@dataclass(frozen=True, eq=False)
class PaddedSignal:
    """A signal extended to alpha*N samples with a zero tail (ref/baseline.py:24-54)."""

    samples: np.ndarray
    original_n: int
    duration: float

    def __post_init__(self):
        arr = np.array(self.samples, dtype=np.complex128)
        if arr.ndim != 1 or not 1 <= self.original_n <= arr.size:
            raise ValueError(f"padded length {arr.shape} incompatible with original N={self.original_n}")
        if np.any(arr[self.original_n:] != 0):
            raise ValueError("padding tail must be exactly zero")
        if not self.duration > 0:
            raise ValueError(f"duration must be positive, got {self.duration}")
        arr.setflags(write=False)
        object.__setattr__(self, "samples", arr)

    def __len__(self) -> int:
        return self.samples.size

    def as_signal(self) -> Signal:
        return Signal(self.samples, self.duration)


def zero_pad(signal: Signal, alpha: DenseFactor) -> PaddedSignal:
    """Extend to alpha*N samples with zeros, alpha >= 1 (ref/baseline.py:57-64)."""
    n, m = validate_pair(len(signal), alpha)
    if alpha.p < alpha.q:
        raise ValueError(f"zero-padding needs alpha >= 1, got {alpha}")
    padded = np.zeros(m, dtype=np.complex128)
    padded[:n] = signal.samples
    return PaddedSignal(padded, n, signal.duration * (alpha.p / alpha.q))


def standard_fft(samples, duration: float = 1.0, counter: OpCounter | None = None) -> Spectrum:
    """Ordinary FFT = the α-FFT at density 1 (ref/baseline.py:67-81)."""
    if isinstance(samples, PaddedSignal):
        signal = samples.as_signal()
    elif isinstance(samples, Signal):
        signal = samples
    else:
        signal = Signal(np.asarray(samples), duration)
    method = "fft" if (len(signal) & (len(signal) - 1)) == 0 else "chirp"
    return alpha_fft(signal, plan(len(signal), DenseFactor(1), method=method), counter)


def aliased_reconstruct(signal: Signal, alpha: DenseFactor) -> np.ndarray:
    """x'_n = Σ_k x_{n+k*alpha*N}, period M, alpha < 1 (ref/baseline.py:84-97), folded on the GPU."""
    n, m = validate_pair(len(signal), alpha)
    if alpha.p >= alpha.q:
        raise ValueError(f"alias folding needs alpha < 1, got {alpha}")
    torch = _torch()
    dev = _default_device()
    k = -(-n // m)
    x = torch.zeros(k * m, dtype=torch.complex128, device=f"cuda:{dev}")
    x[:n] = torch.from_numpy(np.array(signal.samples)).to(x.device)
    cols = x.view(k, m).t().contiguous()  # row r = the samples with residue r
    folded = torch.empty(m, dtype=torch.complex128, device=x.device)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().asx_block_sum(cols.data_ptr(), folded.data_ptr(), m, k, _lib.ASX_C128, st),
               "block_sum")
    return folded[torch.arange(n, device=x.device) % m].cpu().numpy()


__all__ = ["naive_inverse", "orthogonality_kernel", "PaddedSignal", "zero_pad", "standard_fft",
           "aliased_reconstruct"]
