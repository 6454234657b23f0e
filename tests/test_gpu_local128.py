"""GPU parity of the P = 8192 complex128 chirp kernel with group-local
exchanges (csrc/asx_chirp_local128.cuh, BASELINE config 1b) off the BASELINE
shape: ragged N and M, non-dyadic alpha, real input, batches that do not
divide the grid, strided rows -- against the CPU oracle (oracle.py:37-47
restated) and against the Stockham engine it replaces (ASX_NO_LOCAL=1)."""

import os

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
VARIANT_CL128 = 6  # asx_last_launch: k_chirp_local128


@pytest.fixture(scope="module")
def asx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2403_16665_b200 as asx

    return asx


def last_variant():
    import ctypes

    from paper_2403_16665_b200 import _lib

    v = [ctypes.c_int() for _ in range(4)]
    _lib.lib().asx_last_launch(*[ctypes.byref(c) for c in v])
    return v[3].value >> 1


def make_plan(asx, n, a, d, m, real, legacy=False):
    old = os.environ.get("ASX_NO_LOCAL")
    os.environ["ASX_NO_LOCAL"] = "1" if legacy else "0"
    try:
        return asx.plan(n, asx.DenseFactor(d, a), m=m, dtype="complex128", method="chirp", real_input=real)
    finally:
        if old is None:
            del os.environ["ASX_NO_LOCAL"]
        else:
            os.environ["ASX_NO_LOCAL"] = old


CASES = [
    # n, a, d, m, real, batch        (P = nextpow2(n + m - 1) = 8192 in all)
    (4096, 1, 10, 4096, False, 149),  # config-1b shape, one CTA gets two signals
    (2500, 3, 7, 4000, False, 150),   # ragged N and M, non-dyadic alpha
    (4096, 1, 1, 4096, True, 5),      # alpha = 1 (plain DFT), real input
    (2049, 5, 13, 2100, False, 1),    # odd sizes, single signal
]


@pytest.mark.parametrize("n,a,d,m,real,batch", CASES)
def test_local128_vs_oracle_and_engine(asx, n, a, d, m, real, batch):
    import torch

    rng = np.random.default_rng(n + 13 * m + batch)
    x = np.stack([orc.unit_disk(rng, n) for _ in range(batch)])
    if real:
        x = x.real.copy()
    xt = torch.from_numpy(x).cuda()
    p = make_plan(asx, n, a, d, m, real)
    assert p.fft_size == 8192
    got = p.execute(xt)
    torch.cuda.synchronize()
    assert last_variant() == VARIANT_CL128, "the group-local complex128 chirp kernel did not run"
    legacy = make_plan(asx, n, a, d, m, real, legacy=True).execute(xt)
    torch.cuda.synchronize()
    assert last_variant() != VARIANT_CL128
    got = got.cpu().numpy()
    idx = sorted({0, batch - 1, batch // 2})
    want = orc.direct(x[idx].astype(np.complex128), a, d, m)
    assert orc.rel_err(got[idx], want) <= TOL64
    assert orc.rel_err(got, legacy.cpu().numpy()) <= TOL64


def test_local128_strided_rows(asx):
    import torch

    rng = np.random.default_rng(5)
    big = np.stack([orc.unit_disk(rng, 4500) for _ in range(3)])
    view = torch.from_numpy(big).cuda()[:, 3:4099]  # row stride 4500 elements
    p = make_plan(asx, 4096, 1, 10, 4096, False)
    got = p.execute(view).cpu().numpy()
    assert last_variant() == VARIANT_CL128
    want = orc.direct(big[:, 3:4099], 1, 10, 4096)
    assert orc.rel_err(got, want) <= TOL64
