"""CPU restatement of the reference α-DFT / α-FFT — TEST INFRASTRUCTURE ONLY.

This module is the parity oracle.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it, and
there only as the checker or as the timed reference CPU path.  The product
(``paper_2403_16665_b200``) never imports it and has no CPU fallback.

It restates, in batched numpy, the reference package ``alpha-spectra``
(``/root/reference/pkg/src/alpha_spectra``; cited below as ``ref/<file>:<line>``):

* ``direct``      — ref/oracle.py:21-47 (``roots_of_unity``, ``_reduced_product``)
                    and ref/oracle.py:26-34 (``dft_matrix``): one table of L-th roots
                    of unity indexed by the exactly reduced integer exponent.  The
                    reference table is the (alpha*N)-th roots and the exponent
                    ``(m*n) mod M_ref``; here α = a/d is the BASELINE α
                    (= 1/alpha_ref), the table holds the (d*N)-th roots
                    and the exponent is ``(a*m*n) mod (d*N)``, which is identical for
                    every α the reference accepts and also defines the α it rejects
                    (BASELINE config 3, α = 37/100).
* ``alpha_fft``   — ref/fastpath.py:162-181 (``transform_samples``): the
                    level-synchronous even/odd recursion with the ref/fastpath.py:104-109
                    twiddle tables and the ref/fastpath.py:130-151 ``combine`` butterfly,
                    batched over rows; the SINGLE_SAMPLE leaf (ref/fastpath.py:166-169)
                    is generalised to any integer density r (the reference requires a
                    power of two, ref/fastpath.py:97-101), the BLOCK_SUM leaf is
                    ref/fastpath.py:170-174.
* ``combine`` / ``leaf_block_sum`` — ref/fastpath.py:130-151 / :154-159.
* ``predicted_mults`` / ``predicted_adds`` — ref/fastpath.py:113-127.
* ``rel_err``     — the reference's error metric max|ΔX| / max|X| per signal
                    (ref/verify.py:75-77, ref/tests/test_acceptance.py:70-72).

Pinned against the reference itself: ``tests/golden/make_golden.py`` imports
the reference read-only and records its outputs in ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks every function here against them.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

_BLOCK_ROWS = 512  # ref/oracle.py:18 — bound the int64 exponent block


def reduce_alpha(a: int, d: int) -> tuple[int, int]:
    g = math.gcd(a, d)
    return a // g, d // g


def alpha_from_decimal(text: str) -> tuple[int, int]:
    """BASELINE α given as a decimal ('0.37', '1/16') -> reduced (a, d)."""
    fr = Fraction(text)
    return fr.numerator, fr.denominator


def roots(L: int, sign: int = -1) -> np.ndarray:
    """w[j] = exp(sign*2πi j/L), j < L (ref/oracle.py:21-23)."""
    return np.exp(sign * 2j * np.pi * np.arange(L) / L)


def exponent_block(rows: np.ndarray, cols: np.ndarray, a: int, L: int) -> np.ndarray:
    """(a*m*n) mod L in exact integer arithmetic (ref/oracle.py:44-45)."""
    am = (a * rows.astype(np.int64)) % L
    return (am[:, None] * cols.astype(np.int64)[None, :]) % L


def dft_matrix(n: int, a: int, d: int, m: int) -> np.ndarray:
    """W[m, n] = exp(-2πi ((a m n) mod dN)/(dN)) (ref/oracle.py:26-34)."""
    a, d = reduce_alpha(a, d)
    L = d * n
    table = roots(L)
    return table[exponent_block(np.arange(m), np.arange(n), a, L)]


def direct(x: np.ndarray, a: int, d: int, m: int) -> np.ndarray:
    """Direct α-DFT of every row of x (B, N) -> (B, m) complex128.

    Row blocks of _BLOCK_ROWS output bins, exact exponent reduction, then a
    BLAS product, as ref/oracle.py:37-47 does per signal.
    """
    x = np.atleast_2d(np.asarray(x, dtype=np.complex128))
    n = x.shape[1]
    a, d = reduce_alpha(a, d)
    L = d * n
    table = roots(L)
    cols = np.arange(n)
    out = np.empty((x.shape[0], m), dtype=np.complex128)
    for start in range(0, m, _BLOCK_ROWS):
        stop = min(start + _BLOCK_ROWS, m)
        w = table[exponent_block(np.arange(start, stop), cols, a, L)]
        out[:, start:stop] = x @ w.T
    return out


def plan_twiddles(m_ref: int, depth: int) -> list[np.ndarray]:
    """Twiddle table k serves merges of output length m_ref >> k (ref/fastpath.py:104-109)."""
    tables = []
    for k in range(depth):
        size = m_ref >> k
        tables.append(np.exp(-2j * np.pi * np.arange(size // 2) / size))
    return tables


def combine(y: np.ndarray, z: np.ndarray, tw: np.ndarray) -> np.ndarray:
    """[y + w z, y - w z] along the last axis (ref/fastpath.py:130-151)."""
    y = np.asarray(y)
    z = np.asarray(z)
    if y.shape != z.shape:
        raise ValueError(f"half-spectra differ in shape: {y.shape} vs {z.shape}")
    if y.shape[-1] != np.shape(tw)[-1]:
        raise ValueError("twiddle table length does not match half-spectrum length")
    t = tw * z
    return np.concatenate([y + t, y - t], axis=-1)


def leaf_block_sum(block: np.ndarray) -> complex:
    """Plain sum of a sample block (ref/fastpath.py:154-159)."""
    return complex(np.asarray(block, dtype=np.complex128).sum())


def alpha_fft(x: np.ndarray, a: int, d: int, m: int | None = None) -> np.ndarray:
    """α-FFT of every row of x (B, N) at α = a/d; returns (B, m) complex128.

    Supported exactly where the generalised reference recursion is defined:
    α = 1/r (alpha_ref = r integer, SINGLE_SAMPLE leaf) with N a power of two,
    or α = q (alpha_ref = 1/q, BLOCK_SUM leaf) with N/q a power of two.
    Bins past the full spectrum M_ref wrap periodically (W^(m+M_ref) = W^m).
    """
    x = np.atleast_2d(np.asarray(x, dtype=np.complex128))
    bsz, n = x.shape
    a, d = reduce_alpha(a, d)
    if a == 1:
        r = d
        if n & (n - 1):
            raise ValueError("alpha_fft oracle needs power-of-two N")
        m_ref = r * n
        depth = n.bit_length() - 1
        # leaf: row j is the r-bin sub-spectrum of x[j::N] == [x_j] (ref/fastpath.py:166-169)
        level = np.broadcast_to(x[:, :, None], (bsz, n, r))
    elif d == 1:
        q = a
        if n % q or ((n // q) & (n // q - 1)):
            raise ValueError("alpha_fft oracle needs N/q a power of two")
        m_ref = n // q
        depth = m_ref.bit_length() - 1
        # leaf: row c is the 1-bin sub-spectrum of x[c::M], its block sum (ref/fastpath.py:170-174)
        level = x.reshape(bsz, -1, m_ref).sum(axis=1)[:, :, None]
    else:
        raise ValueError("alpha_fft oracle needs alpha = 1/r or alpha = q")
    tables = plan_twiddles(m_ref, depth)
    for k in range(depth - 1, -1, -1):  # ref/fastpath.py:175-180
        half = level.shape[1] // 2
        level = combine(level[:, :half], level[:, half:], tables[k])
    full = np.array(level, dtype=np.complex128).reshape(bsz, m_ref)
    if m is None:
        return full
    idx = np.arange(m) % m_ref
    return full[:, idx]


def predicted_mults(n: int, m_ref: int) -> int:
    """(M/2) * log2(min(N, M)) (ref/fastpath.py:113-121)."""
    depth = min(n, m_ref).bit_length() - 1
    return (m_ref // 2) * depth


def predicted_adds(n: int, m_ref: int) -> int:
    """M * depth + block-sum leaf adds (ref/fastpath.py:124-127)."""
    depth = min(n, m_ref).bit_length() - 1
    return m_ref * depth + (n - m_ref if m_ref < n else 0)


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """Worst per-signal max|ΔX| / max|X| over the batch (ref/verify.py:75-77)."""
    got = np.atleast_2d(np.asarray(got, dtype=np.complex128))
    want = np.atleast_2d(np.asarray(want, dtype=np.complex128))
    if got.shape != want.shape:
        raise ValueError(f"shape mismatch {got.shape} vs {want.shape}")
    if got.size == 0:
        return 0.0
    scale = np.maximum(np.max(np.abs(want), axis=1), 1e-300)
    return float(np.max(np.max(np.abs(got - want), axis=1) / scale))


def unit_disk(rng: np.random.Generator, n: int) -> np.ndarray:
    """n complex samples uniform on the unit disk (ref/verify.py:42-46 convention)."""
    radius = np.sqrt(rng.uniform(0.0, 1.0, n))
    angle = rng.uniform(0.0, 2.0 * np.pi, n)
    return radius * np.exp(1j * angle)
