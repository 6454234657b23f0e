"""GPU parity of the 32-values-per-thread chirp kernel (csrc/asx_chirp_r32.cuh:
P = 16384 complex64, N, M <= 8192 -- the config-4 hot kernel) off the BASELINE
shape: ragged N and M, real input, batches that do not divide the grid,
strided input and output rows -- against the CPU oracle (oracle.py:37-47
restated), against the 16-values-per-thread kernel (ASX_NO_R32=1,
k_chirp_local) and, signal by signal, against the complex128 GPU path."""

import os

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu

TOL32 = 2e-5
VARIANT_R32 = 14  # asx_last_launch: k_chirp_r32
VARIANT_LOCAL = 2  # asx_last_launch: k_chirp_local


@pytest.fixture(scope="module")
def asx():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("GPU tests need a CUDA device")
    import paper_2403_16665_b200 as asx

    return asx


def last_variant():
    import ctypes

    from paper_2403_16665_b200 import _lib

    v = [ctypes.c_int() for _ in range(4)]
    _lib.lib().asx_last_launch(*[ctypes.byref(c) for c in v])
    return v[3].value >> 1


def make_plan(asx, n, a, d, m, real=False, r32=True, dtype="complex64"):
    old = os.environ.get("ASX_NO_R32")
    os.environ["ASX_NO_R32"] = "0" if r32 else "1"
    try:
        return asx.plan(n, asx.DenseFactor(d, a), m=m, dtype=dtype, method="chirp", real_input=real)
    finally:
        if old is None:
            del os.environ["ASX_NO_R32"]
        else:
            os.environ["ASX_NO_R32"] = old


CASES = [
    # n, a, d, m, real, batch        (P = nextpow2(n + m - 1) = 16384 in all)
    (8192, 1, 8, 8192, False, 149),  # config-4 shape, one CTA gets two signals
    (8192, 1, 8, 8192, False, 1),    # single signal
    (5000, 3, 7, 7000, False, 150),  # ragged N and M, non-dyadic alpha
    (8192, 1, 1, 8192, True, 5),     # alpha = 1 (plain DFT), real input
    (4097, 5, 13, 4100, False, 3),   # odd sizes
    (8191, 37, 100, 8192, False, 5), # config-3 alpha on long signals, N odd
]


@pytest.mark.parametrize("n,a,d,m,real,batch", CASES)
def test_r32_kernel_vs_oracle_and_local(asx, n, a, d, m, real, batch):
    import torch

    rng = np.random.default_rng(n + 17 * m + batch)
    x = np.stack([orc.unit_disk(rng, n) for _ in range(batch)])
    if real:
        x = x.real.copy()
    x = x.astype(np.float32 if real else np.complex64)
    xt = torch.from_numpy(x).cuda()
    p = make_plan(asx, n, a, d, m, real)
    assert p.fft_size == 16384
    got = p.execute(xt)
    torch.cuda.synchronize()
    assert last_variant() == VARIANT_R32, "the 32-values-per-thread kernel did not run"
    local = make_plan(asx, n, a, d, m, real, r32=False).execute(xt)
    torch.cuda.synchronize()
    assert last_variant() == VARIANT_LOCAL
    got = got.cpu().numpy()
    idx = sorted({0, batch - 1, batch // 2})
    want = orc.direct(x[idx].astype(np.complex128), a, d, m)
    assert orc.rel_err(got[idx], want) <= TOL32
    assert orc.rel_err(got, local.cpu().numpy()) <= 2 * TOL32
    # every signal against the complex128 GPU path on the same inputs
    x128 = xt.to(torch.float64 if real else torch.complex128)
    ref = make_plan(asx, n, a, d, m, real, dtype="complex128").execute(x128).cpu().numpy()
    err = np.abs(got - ref).max(axis=1) / np.abs(ref).max(axis=1)
    assert err.max() <= TOL32, err.max()


def test_r32_kernel_strided_rows(asx):
    import torch

    rng = np.random.default_rng(7)
    big = np.stack([orc.unit_disk(rng, 9000) for _ in range(5)]).astype(np.complex64)
    view = torch.from_numpy(big).cuda()[:, 100:8292]  # input row stride 9000 (no TMA staging)
    p = make_plan(asx, 8192, 1, 8, 8192)
    outbuf = torch.full((5, 9001), 7 + 7j, dtype=torch.complex64, device="cuda")
    out = outbuf[:, 3:8195]  # output row stride 9001, odd offset
    p.execute(view, out=out)
    torch.cuda.synchronize()
    assert last_variant() == VARIANT_R32
    want = orc.direct(big[:, 100:8292].astype(np.complex128), 1, 8, 8192)
    assert orc.rel_err(out.cpu().numpy(), want) <= TOL32
    guard = outbuf.cpu().numpy()
    assert np.all(guard[:, :3] == 7 + 7j) and np.all(guard[:, 8195:] == 7 + 7j)  # nothing outside the rows


def test_r32_kernel_repeatable(asx):
    """Bit-for-bit repeat determinism, alone and with a memory-heavy kernel
    perturbing the schedule (a missing barrier around the CTA-wide or the
    warp-local exchange would make the result depend on warp timing)."""
    import torch

    rng = np.random.default_rng(11)
    x = torch.from_numpy(np.stack([orc.unit_disk(rng, 8192) for _ in range(600)]).astype(np.complex64)).cuda()
    p = make_plan(asx, 8192, 1, 8, 8192)
    first = p.execute(x).clone()
    noise = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    for _ in range(5):
        with torch.cuda.stream(side):
            noise.normal_()
        again = p.execute(x)
        torch.cuda.synchronize()
        assert last_variant() == VARIANT_R32
        assert torch.equal(torch.view_as_real(first), torch.view_as_real(again))
