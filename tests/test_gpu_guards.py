"""Memory-safety and race checks of the hot kernels without compute-sanitizer
(closed on this GPU pool: runs under it left GPUs needing a reset).

* Guard bands (memcheck's job): inputs and outputs live inside larger
  buffers filled with a sentinel; after the launch every byte outside the
  transform's rows / bins must still hold the sentinel and the input must be
  unchanged -- on ragged N and M, odd batches, partial tiles and strided
  (unaligned) rows, the cases where an off-by-one store would land.
* Repeat determinism (racecheck / synccheck's job): the kernels exchange
  data through shared memory behind split-phase mbarriers, named barriers and
  "each thread rewrites exactly the slots it read" local exchanges, fetch
  rows by TMA and keep tables in tensor memory.  A missing barrier makes the
  result depend on warp timing, so every kernel runs many times -- alone and
  with a concurrent memory-heavy kernel on another stream perturbing its
  schedule -- and must reproduce the first result bit for bit, and match the
  CPU oracle.
"""

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu

# (label, n, alpha_b = a/d, m, dtype, method, batch) -> the kernel it launches
KERNELS = [
    ("k_chirp_r32", 8192, 1, 8, 8192, "complex64", "chirp", 300),
    ("k_chirp_r32 ragged", 6000, 1, 8, 7001, "complex64", "chirp", 151),
    ("k_afft_local", 4096, 1, 2, 4096, "complex128", "fft", 300),
    ("k_afft_local M < N", 4096, 1, 2, 3001, "complex128", "fft", 151),
    ("k_chirp_local128", 4096, 1, 10, 4096, "complex128", "chirp", 300),
    ("k_chirp_local128 ragged", 3001, 1, 10, 4000, "complex128", "chirp", 151),
    ("k_direct_tc", 256, 37, 100, 256, "complex64", "direct", 1000),
    ("k_direct_tc ragged tile", 96, 2, 3, 256, "complex64", "direct", 131),
    ("k_fft_persist alpha-FFT FP64 / c64 I/O", 1024, 1, 4, 1024, "complex64", "fft", 301),
    ("k_fft_persist alpha-FFT block-sum leaf", 1024, 4, 1, 256, "complex128", "fft", 77),
    ("k_fft_persist chirp warp teams", 256, 37, 100, 256, "complex64", "chirp", 1001),
    ("four-step chirp", 8192, 1, 8, 8192, "complex128", "chirp", 2),
    ("four-step alpha-FFT", 16384, 1, 2, 16384, "complex128", "fft", 2),
]
TOL = {"complex64": 2e-5, "complex128": 1e-10}


@pytest.fixture(scope="module")
def env():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2403_16665_b200 as asx

    return torch, asx


def _signals(n, batch, dtype, seed):
    rng = np.random.default_rng(seed)
    x = np.stack([orc.unit_disk(rng, n) for _ in range(batch)])
    return x.astype(np.complex64 if dtype == "complex64" else np.complex128)


@pytest.mark.parametrize("case", KERNELS, ids=[k[0] for k in KERNELS])
@pytest.mark.parametrize("pad", [0, 3])
def test_guard_bands(env, case, pad):
    torch, asx = env
    label, n, a, d, m, dtype, method, batch = case
    cdt = getattr(torch, dtype)
    x = _signals(n, batch, dtype, n + m)
    sentinel = complex(np.float32(-7.25e3), np.float32(3.5e-3))
    # rows of n (+ pad) inside a buffer with one guard row before and after
    xin = torch.full((batch + 2, n + pad), sentinel, dtype=cdt, device="cuda")
    xin[1:batch + 1, :n] = torch.from_numpy(x).cuda()
    xin_before = xin.clone()
    out = torch.full((batch + 2, m + pad), sentinel, dtype=cdt, device="cuda")
    p = asx.plan(n, asx.DenseFactor(d, a), m=m, dtype=dtype, method=method)
    p.execute(xin[1:batch + 1, :n], out=out[1:batch + 1, :m])
    torch.cuda.synchronize()
    assert torch.equal(xin, xin_before), "input modified"
    o = out.cpu().numpy()
    guard = np.ones(o.shape, bool)
    guard[1:batch + 1, :m] = False
    assert np.all(o[guard] == np.complex64(sentinel) if dtype == "complex64" else o[guard] == sentinel), \
        f"{label}: store outside the output rows"
    idx = np.unique(np.linspace(0, batch - 1, 5).astype(int))
    want = orc.direct(x[idx].astype(np.complex128), a, d, m)
    assert orc.rel_err(o[1:batch + 1, :m][idx], want) <= TOL[dtype], label


@pytest.mark.parametrize("case", KERNELS, ids=[k[0] for k in KERNELS])
def test_repeat_determinism_under_perturbation(env, case):
    torch, asx = env
    label, n, a, d, m, dtype, method, batch = case
    x = torch.from_numpy(_signals(n, batch, dtype, 99)).cuda()
    p = asx.plan(n, asx.DenseFactor(d, a), m=m, dtype=dtype, method=method)
    first = p.execute(x).clone()
    noise_src = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    noise_dst = torch.empty_like(noise_src)
    side = torch.cuda.Stream()
    reps = 6 if "four-step" in label else 20
    for i in range(reps):
        if i % 2:
            with torch.cuda.stream(side):  # a concurrent HBM-heavy kernel shifts the schedule
                for _ in range(3):
                    noise_dst.copy_(noise_src)
        y = p.execute(x)
        assert torch.equal(y, first), f"{label}: run {i} differs from run 0"
    torch.cuda.synchronize()
