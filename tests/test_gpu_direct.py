"""GPU parity of the direct α-DFT (ref/oracle.py:37-67 `naive_forward`, the
matrix form with exactly reduced exponents) on both of its kernels: the
64 x 64 tiled contraction (k_direct, batches above 8) and the per-bin
matrix-vector kernel for a handful of signals (k_direct_small) -- against the
CPU oracle, complex64 and complex128, ragged N and M, non-dyadic alpha."""

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def asx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2403_16665_b200 as asx

    return asx


@pytest.mark.parametrize("batch", [1, 3, 8, 9, 70])
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-10), ("complex64", 2e-5)])
@pytest.mark.parametrize("n,a,d,m", [(256, 37, 100, 256), (300, 2, 3, 257), (1024, 1, 4, 1024)])
def test_direct_vs_oracle(asx, batch, dtype, tol, n, a, d, m):
    import torch

    rng = np.random.default_rng(batch + 7 * n + m)
    x = np.stack([orc.unit_disk(rng, n) for _ in range(batch)])
    xin = x.astype(np.complex64).astype(np.complex128) if dtype == "complex64" else x
    p = asx.plan(n, asx.DenseFactor(d, a), m=m, dtype=dtype, method="direct")
    got = p.execute(torch.from_numpy(xin.astype(dtype)).cuda()).cpu().numpy()
    assert got.shape == (batch, m)
    assert orc.rel_err(got, orc.direct(xin, a, d, m)) <= tol
