"""CPU emulation of the tensor-core direct form's arithmetic (k_direct_tc,
csrc/asx_direct_tc.cuh): per-signal power-of-two scaling, fp16 hi/lo splits
of the signal and of W = exp(-2 pi i (a m n mod dN) / dN) (ref/oracle.py:37-47
exact reduction), and Re X = Ar Wr - Ai Wi, Im X = Ar Wi + Ai Wr as sums of
A_hi B_hi + A_hi B_lo + A_lo B_hi products.  Checks, against the oracle on
BASELINE config-3 signals, that this three-product scheme meets the
complex64 bound (2e-5 of max|X|) and that one fp16 product per term does not
-- the reason the kernel issues three MMAs per real product.

`_emulate` rounds every GEMM once; `_emulate_stepwise` follows the kernel's
accumulation instead: one fp32 accumulator update per 16-sample MMA in the
kernel's issue order (csrc/asx_direct_tc.cuh, the `step` lambda), each update
rounded toward zero (tensor-core accumulation is not round-to-nearest; toward
zero is the conservative model).  It is checked at N = 256 (config 3) and at
N = 1024, the largest N the plan gives to k_direct_tc."""

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


def _rtz32(v):
    """float64 -> float32 rounded toward zero."""
    f = v.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(v)
    return np.where(over, np.nextafter(f, np.float32(0)), f).astype(np.float32)


def _emulate_stepwise(x, a, d, m):
    n = x.shape[1]
    ph = (a * np.arange(m)[:, None] * np.arange(n)[None, :]) % (d * n)
    w = np.exp(-2j * np.pi * ph / (d * n)) * 256.0
    xr, xi = x.real.astype(np.float64), x.imag.astype(np.float64)
    mx = np.maximum(np.abs(xr).max(axis=1), np.abs(xi).max(axis=1))
    s = 2.0 ** (10 - np.floor(np.log2(np.where(mx > 0, mx, 1.0))))
    (arh, arl), (aih, ail) = _split(xr * s[:, None]), _split(xi * s[:, None])
    (wrh, wrl), (wih, wil) = _split(w.real), _split(w.imag)
    re = np.zeros((x.shape[0], m), np.float32)
    im = np.zeros((x.shape[0], m), np.float32)

    def upd(acc, a_, b_, k, sign=1.0):  # one 128 x N x 16 MMA: exact products, one truncated accumulate
        part = a_[:, k:k + 16] @ b_[:, k:k + 16].T
        return _rtz32(acc.astype(np.float64) + sign * part)

    for c in range(0, n, 32):           # K chunk
        for k in (c, c + 16):           # part 0 (Wr): Re += Ar Wr, Im += Ai Wr
            re, im = upd(re, arh, wrh, k), upd(im, aih, wrh, k)
            re, im = upd(re, arh, wrl, k), upd(im, aih, wrl, k)
            re, im = upd(re, arl, wrh, k), upd(im, ail, wrh, k)
        for k in (c, c + 16):           # part 1 (Wi): Re -= Ai Wi, Im += Ar Wi
            re, im = upd(re, aih, wih, k, -1.0), upd(im, arh, wih, k)
            re, im = upd(re, aih, wil, k, -1.0), upd(im, arh, wil, k)
            re, im = upd(re, ail, wih, k, -1.0), upd(im, arl, wih, k)
    return (re.astype(np.float64) + 1j * im.astype(np.float64)) / (s[:, None] * 256.0)


def test_stepwise_truncating_accumulation_meets_bound_up_to_the_plan_cap():
    w = signals.WORKLOADS["3"]
    x = signals.generate(w, 0, 64).astype(np.complex64)
    want = orc.direct(x.astype(np.complex128), 37, 100, 256)
    assert orc.rel_err(_emulate_stepwise(x, 37, 100, 256), want) <= TOL / 2
    # N = 1024 (asx_api.cu caps the tensor-core form there): tones + noise and unit-disk noise
    rng = np.random.default_rng(5)
    n = 1024
    t = np.arange(n)
    tones = np.stack([sum(rng.uniform(0.1, 1) * np.exp(2j * np.pi * rng.uniform(0, n / 2) * t / n) for _ in range(2))
                      + 0.01 * (rng.standard_normal(n) + 1j * rng.standard_normal(n)) for _ in range(16)])
    noise = np.stack([orc.unit_disk(rng, n) for _ in range(16)])
    for xs in (tones, noise):
        xs = xs.astype(np.complex64)
        want = orc.direct(xs.astype(np.complex128), 37, 100, 256)
        assert orc.rel_err(_emulate_stepwise(xs, 37, 100, 256), want) <= TOL


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
