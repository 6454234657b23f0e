"""GPU parity of the complex128 group-local α-FFT kernel (csrc/asx_afft_local.cuh,
config 1a: N = 4096, α = 1/2, the reference's DenseFactor(2) recursion,
ref/fastpath.py:162-181) off the BASELINE shape: M below N (odd, and below
one residue), batches that do not divide the grid, a single signal, strided
rows, and the fall-back to the Stockham engine for rows TMA cannot stage --
against the CPU oracle and against that engine (ASX_NO_AFFT_LOCAL=1)."""

import os

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
VARIANT_AFL = 4  # asx_last_launch: k_afft_local


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


def make_plan(asx, m, legacy=False):
    old = os.environ.get("ASX_NO_AFFT_LOCAL")
    os.environ["ASX_NO_AFFT_LOCAL"] = "1" if legacy else "0"
    try:
        return asx.plan(4096, asx.DenseFactor(2), m=m, dtype="complex128", method="fft")
    finally:
        if old is None:
            del os.environ["ASX_NO_AFFT_LOCAL"]
        else:
            os.environ["ASX_NO_AFFT_LOCAL"] = old


@pytest.mark.parametrize("m,batch", [(4096, 149), (4095, 150), (3001, 1), (1500, 300), (1, 2)])
def test_afft_local_vs_oracle_and_engine(asx, m, batch):
    import torch

    rng = np.random.default_rng(m + 31 * batch)
    x = np.stack([orc.unit_disk(rng, 4096) for _ in range(batch)])
    xt = torch.from_numpy(x).cuda()
    got = make_plan(asx, m).execute(xt)
    torch.cuda.synchronize()
    assert last_variant() == VARIANT_AFL, "the group-local alpha-FFT kernel did not run"
    legacy = make_plan(asx, m, legacy=True).execute(xt)
    torch.cuda.synchronize()
    assert last_variant() != VARIANT_AFL
    got = got.cpu().numpy()
    idx = sorted({0, batch - 1, batch // 2})
    want = orc.alpha_fft(x[idx], 1, 2, m)  # the reference recursion, restated
    assert orc.rel_err(got[idx], want) <= TOL64
    assert orc.rel_err(got, legacy.cpu().numpy()) <= TOL64


def test_afft_local_strided_rows(asx):
    import torch

    rng = np.random.default_rng(11)
    big = np.stack([orc.unit_disk(rng, 4200) for _ in range(5)])
    # row stride 4200 elements (16-byte aligned rows: TMA staging still applies)
    view = torch.from_numpy(big).cuda()[:, 8:4104]
    got = make_plan(asx, 4096).execute(view).cpu().numpy()
    assert last_variant() == VARIANT_AFL
    assert orc.rel_err(got, orc.alpha_fft(big[:, 8:4104], 1, 2, 4096)) <= TOL64


def test_afft_local_output_stride(asx):
    import torch

    rng = np.random.default_rng(12)
    x = np.stack([orc.unit_disk(rng, 4096) for _ in range(3)])
    out = torch.zeros((3, 4500), dtype=torch.complex128, device="cuda")
    make_plan(asx, 4096).execute(torch.from_numpy(x).cuda(), out=out[:, :4096])
    assert last_variant() == VARIANT_AFL
    o = out.cpu().numpy()
    assert orc.rel_err(o[:, :4096], orc.alpha_fft(x, 1, 2, 4096)) <= TOL64
    assert not np.any(o[:, 4096:]), "wrote past the row"


def test_afft_local_not_used_for_real_input(asx):
    import torch

    rng = np.random.default_rng(13)
    x = np.stack([orc.unit_disk(rng, 4096).real for _ in range(2)])
    p = asx.plan(4096, asx.DenseFactor(2), m=4096, dtype="complex128", method="fft", real_input=True)
    got = p.execute(torch.from_numpy(x).cuda()).cpu().numpy()
    assert last_variant() != VARIANT_AFL
    assert orc.rel_err(got, orc.alpha_fft(x.astype(np.complex128), 1, 2, 4096)) <= TOL64
