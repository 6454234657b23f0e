"""BASELINE.json workloads and their seeded synthetic signals.

There is no public dataset for this path; the five BASELINE
configs are restated here as ``WORKLOADS`` and their signals are sums of
tones plus Gaussian noise drawn from numpy PCG64 with one stream per signal,
``default_rng([seed, index])``, so every shard of a batch is reproducible on
its own.  Per signal and per component (real part, then imaginary part for
complex configs) the draw order is: amplitudes A[K], frequencies f[K],
phases φ[K], noise ε[N]; x_n = Σ_k A_k cos(2π f_k n/N + φ_k) + ε_n, generated
in float64 and then cast to the config dtype.  Tone synthesis for large
batches runs on the GPU from the host-drawn parameters and noise.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from fractions import Fraction

import numpy as np


@dataclass(frozen=True)
class Workload:
    key: str
    n: int
    alpha: Fraction  # BASELINE α: X_m = Σ x_n exp(-2πi α m n / N)
    m: int
    batch: int
    dtype: str  # complex64 | complex128 (arithmetic and output type)
    real: bool  # real-valued input samples
    tones: int
    amp: tuple
    freq: tuple  # (lo, hi) uniform, or ("midbin", lo, hi): integer in [lo, hi) + 0.5
    sigma: float
    seed: int
    note: str = ""

    @property
    def density(self):
        from .core import density_for_alpha

        return density_for_alpha(self.alpha)

    def bytes_alg(self, batch=None) -> int:
        """One read of the input and one write of the output."""
        b = self.batch if batch is None else batch
        re = 4 if self.dtype == "complex64" else 8
        in_b = re if self.real else 2 * re
        return b * (self.n * in_b + self.m * 2 * re)

    def flops_alg(self, batch=None) -> int:
        """Reference closed-form α-FFT flops 6*mults + 2*adds."""
        b = self.batch if batch is None else batch
        a, d = self.alpha.numerator, self.alpha.denominator
        if (self.n * d) % a:
            return 8 * self.n * self.m * b  # direct form
        m_ref = self.n * d // a
        depth = min(self.n, m_ref).bit_length() - 1
        mults = (m_ref // 2) * depth
        adds = m_ref * depth + (self.n - m_ref if m_ref < self.n else 0)
        return b * (6 * mults + 2 * adds)


def _wl(key, n, alpha, m, batch, dtype, real, tones, amp, freq, sigma, seed, note):
    return Workload(key, n, Fraction(alpha), m, batch, dtype, real, tones, amp, freq, sigma, seed, note)


WORKLOADS = {
    "0": _wl("0", 1024, "1/4", 1024, 1, "complex128", True, 3, (0.5, 2.0), (10.0, 502.0), 0.1, 0,
             "single real f64 signal, direct + fft"),
    "1a": _wl("1a", 4096, "1/2", 4096, 4096, "complex128", False, 5, (0.5, 2.0), (10.0, 2038.0), 0.05, 1,
              "batch 4096 x 4096 c128, alpha 0.5"),
    "1b": _wl("1b", 4096, "1/10", 4096, 4096, "complex128", False, 5, (0.5, 2.0), (10.0, 2038.0), 0.05, 1,
              "batch 4096 x 4096 c128, alpha 0.1 (same signals as 1a)"),
    "2": _wl("2", 1 << 22, "1/16", 1 << 22, 1, "complex128", True, 8, (0.5, 2.0), ("midbin", 10, (1 << 22) // 16 - 10),
             0.2, 2, "single real f64 signal N=2^22"),
    "3": _wl("3", 256, "37/100", 256, 262144, "complex64", False, 2, (0.1, 1.0), (10.0, 118.0), 0.01, 3,
             "short-signal large-batch direct, non-dyadic alpha"),
    "4": _wl("4", 8192, "1/8", 8192, 65536, "complex64", False, 4, (0.5, 2.0), (0.0, 4096.0), 0.1, 4,
             "multi-GPU batch sweep, sharded over 1/2/4/8"),
}


def _draw(w: Workload, index: int):
    """Per-signal parameters and noise: arrays (C, K) x3 and (C, N), C components."""
    rng = np.random.default_rng([w.seed, index])
    comps = 1 if w.real else 2
    A = np.empty((comps, w.tones))
    F = np.empty((comps, w.tones))
    P = np.empty((comps, w.tones))
    E = np.empty((comps, w.n))
    for c in range(comps):
        A[c] = rng.uniform(w.amp[0], w.amp[1], w.tones)
        if w.freq[0] == "midbin":
            F[c] = rng.integers(w.freq[1], w.freq[2], w.tones) + 0.5
        else:
            F[c] = rng.uniform(w.freq[0], w.freq[1], w.tones)
        P[c] = rng.uniform(0.0, 2.0 * math.pi, w.tones)
        E[c] = rng.normal(0.0, w.sigma, w.n)
    return A, F, P, E


def _draw_many(w: Workload, start: int, count: int, threads: int):
    comps = 1 if w.real else 2
    A = np.empty((count, comps, w.tones))
    F = np.empty_like(A)
    P = np.empty_like(A)
    E = np.empty((count, comps, w.n))

    def fill(i):
        A[i], F[i], P[i], E[i] = _draw(w, start + i)

    if threads > 1 and count > 64:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(fill, range(count), chunksize=max(1, count // (threads * 8))))
    else:
        for i in range(count):
            fill(i)
    return A, F, P, E


def _synth_numpy(w, A, F, P, E):
    t = np.arange(w.n, dtype=np.float64) / w.n
    comps = E + np.einsum("bck,bckn->bcn", A, np.cos(2.0 * math.pi * F[..., None] * t + P[..., None]))
    return comps


def generate(w: Workload, start: int = 0, count: int | None = None, threads: int | None = None) -> np.ndarray:
    """Host signals [start, start+count) of workload w, shape (count, N), config dtype."""
    count = w.batch - start if count is None else count
    threads = threads or min(16, os.cpu_count() or 1)
    A, F, P, E = _draw_many(w, start, count, threads)
    comps = _synth_numpy(w, A, F, P, E)
    if w.real:
        return comps[:, 0].astype(np.float32 if w.dtype == "complex64" else np.float64)
    x = comps[:, 0] + 1j * comps[:, 1]
    return x.astype(np.complex64 if w.dtype == "complex64" else np.complex128)


def generate_device(w: Workload, start: int = 0, count: int | None = None, device="cuda",
                    chunk: int = 1024, threads: int | None = None):
    """Same signals as ``generate`` built into a CUDA tensor (tones synthesised on the GPU)."""
    import torch

    count = w.batch - start if count is None else count
    threads = threads or min(16, os.cpu_count() or 1)
    if w.real:
        out = torch.empty((count, w.n), dtype=torch.float32 if w.dtype == "complex64" else torch.float64,
                          device=device)
    else:
        out = torch.empty((count, w.n), dtype=getattr(torch, w.dtype), device=device)
    t = torch.arange(w.n, dtype=torch.float64, device=device) / w.n
    for c0 in range(0, count, chunk):
        cn = min(chunk, count - c0)
        A, F, P, E = (torch.from_numpy(v).to(device) for v in _draw_many(w, start + c0, cn, threads))
        phase = 2.0 * math.pi * F[..., None] * t + P[..., None]
        comps = E + (A[..., None] * torch.cos(phase)).sum(dim=2)
        if w.real:
            out[c0:c0 + cn] = comps[:, 0].to(out.dtype)
        else:
            out[c0:c0 + cn] = torch.complex(comps[:, 0], comps[:, 1]).to(out.dtype)
    return out
