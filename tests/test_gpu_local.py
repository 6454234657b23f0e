"""GPU parity of the P = 16384 complex64 chirp kernel with group-local
exchanges (csrc/asx_chirp_local.cuh, the config-4 hot kernel) off the
BASELINE shapes: ragged N and M, real input, batches that do not divide the
grid, strided rows -- against the CPU oracle (oracle.py:37-47 restated) and
against the one-exchange-per-pass kernel it replaced (ASX_NO_LOCAL=1)."""

import os

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu

TOL32 = 2e-5


@pytest.fixture(scope="module")
def asx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2403_16665_b200 as asx

    return asx


def last_variant(asx):
    import ctypes

    from paper_2403_16665_b200 import _lib

    v = [ctypes.c_int() for _ in range(4)]
    _lib.lib().asx_last_launch(*[ctypes.byref(c) for c in v])
    return v[3].value >> 1


def make_plan(asx, n, a, d, m, real, legacy=False):
    # ASX_NO_R32=1: the 32-values-per-thread kernel (k_chirp_r32, tests/test_gpu_r32.py) takes
    # these shapes by default; this file pins k_chirp_local, its A/B partner
    old = {k: os.environ.get(k) for k in ("ASX_NO_LOCAL", "ASX_NO_R32")}
    os.environ["ASX_NO_LOCAL"] = "1" if legacy else "0"
    os.environ["ASX_NO_R32"] = "1"
    try:
        return asx.plan(n, asx.DenseFactor(d, a), m=m, dtype="complex64", method="chirp", real_input=real)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


CASES = [
    # n, a, d, m, real, batch        (P = nextpow2(n + m - 1) = 16384 in all)
    (8192, 1, 8, 8192, False, 149),  # config-4 shape, one CTA gets two signals
    (5000, 3, 7, 7000, False, 150),  # ragged N and M, non-dyadic alpha
    (8192, 1, 1, 8192, True, 5),     # alpha = 1 (plain DFT), real input
    (4097, 5, 13, 4100, False, 1),   # odd sizes, single signal
]


@pytest.mark.parametrize("n,a,d,m,real,batch", CASES)
def test_local_kernel_vs_oracle_and_legacy(asx, n, a, d, m, real, batch):
    import torch

    rng = np.random.default_rng(n + 17 * m + batch)
    x = np.stack([orc.unit_disk(rng, n) for _ in range(batch)])
    if real:
        x = x.real.copy()
    xt = torch.from_numpy(x.astype(np.float32 if real else np.complex64)).cuda()
    p = make_plan(asx, n, a, d, m, real)
    assert p.fft_size == 16384
    got = p.execute(xt)
    torch.cuda.synchronize()
    assert last_variant(asx) == 2, "the group-local kernel did not run"
    legacy = make_plan(asx, n, a, d, m, real, legacy=True).execute(xt)
    torch.cuda.synchronize()
    assert last_variant(asx) != 2
    got = got.cpu().numpy()
    # oracle on a sample of signals (complex128, on the complex64-rounded input)
    idx = sorted({0, batch - 1, batch // 2})
    xin = x.astype(np.float32 if real else np.complex64).astype(np.complex128)
    want = orc.direct(xin[idx], a, d, m)
    assert orc.rel_err(got[idx], want) <= TOL32
    assert orc.rel_err(got, legacy.cpu().numpy()) <= 2 * TOL32


def test_local_kernel_strided_rows(asx):
    import torch

    rng = np.random.default_rng(7)
    big = np.stack([orc.unit_disk(rng, 9000) for _ in range(3)]).astype(np.complex64)
    view = torch.from_numpy(big).cuda()[:, 100:8292]  # row stride 9000 (no TMA staging)
    p = make_plan(asx, 8192, 1, 8, 8192, False)
    got = p.execute(view).cpu().numpy()
    assert last_variant(asx) == 2
    want = orc.direct(big[:, 100:8292].astype(np.complex128), 1, 8, 8192)
    assert orc.rel_err(got, want) <= TOL32
