"""CPU emulation of the tensor-core direct form's arithmetic (k_direct_tc,
csrc/asx_direct_tc.cuh): per-signal power-of-two scaling, fp16 hi/lo splits
of the signal and of W = exp(-2 pi i (a m n mod dN) / dN) (ref/oracle.py:37-47
exact reduction), and Re X = Ar Wr - Ai Wi, Im X = Ar Wi + Ai Wr as sums of
A_hi B_hi + A_hi B_lo + A_lo B_hi products.  Checks, against the oracle on
BASELINE config-3 signals, that this three-product scheme meets the
complex64 bound (2e-5 of max|X|) and that one fp16 product per term does not
-- the reason the kernel issues three MMAs per real product."""

import numpy as np

from oracle import alpha_oracle as orc
from paper_2403_16665_b200 import signals

TOL = 2e-5


def _split(v):
    hi = v.astype(np.float16).astype(np.float64)
    return hi, (v - hi).astype(np.float16).astype(np.float64)


def _emulate(x, a, d, m, products):
    n = x.shape[1]
    ph = (a * np.arange(m)[:, None] * np.arange(n)[None, :]) % (d * n)
    w = np.exp(-2j * np.pi * ph / (d * n)) * 256.0  # W_SCALE
    xr, xi = x.real.astype(np.float64), x.imag.astype(np.float64)
    mx = np.maximum(np.abs(xr).max(axis=1), np.abs(xi).max(axis=1))
    s = 2.0 ** (10 - np.floor(np.log2(np.where(mx > 0, mx, 1.0))))  # max |x| into [2^10, 2^11)
    (arh, arl), (aih, ail) = _split(xr * s[:, None]), _split(xi * s[:, None])
    (wrh, wrl), (wih, wil) = _split(w.real), _split(w.imag)

    def gemm(ah, al, bh, bl):
        r = (ah @ bh.T).astype(np.float32)
        if products == 3:
            r = r + (ah @ bl.T).astype(np.float32) + (al @ bh.T).astype(np.float32)
        return r.astype(np.float64)

    re = gemm(arh, arl, wrh, wrl) - gemm(aih, ail, wih, wil)
    im = gemm(arh, arl, wih, wil) + gemm(aih, ail, wrh, wrl)
    return (re + 1j * im) / (s[:, None] * 256.0)


def test_three_fp16_products_meet_complex64_bound():
    w = signals.WORKLOADS["3"]
    x = signals.generate(w, 0, 256).astype(np.complex64)
    want = orc.direct(x.astype(np.complex128), 37, 100, 256)
    assert orc.rel_err(_emulate(x, 37, 100, 256, 3), want) <= TOL / 4
    assert orc.rel_err(_emulate(x, 37, 100, 256, 1), want) > 10 * TOL


def test_scaling_keeps_fp16_in_range():
    rng = np.random.default_rng(1)
    x = np.stack([orc.unit_disk(rng, 256) for _ in range(8)]) * np.array([1e-12, 1e-6, 1, 1e4, 1e12, 3, 5e-3, 7e7])[:, None]
    x = x.astype(np.complex64)
    want = orc.direct(x.astype(np.complex128), 37, 100, 256)
    assert orc.rel_err(_emulate(x, 37, 100, 256, 3), want) <= TOL / 4
