"""GPU parity: every CUDA method against the reference's golden vectors and the
CPU oracle, on the same inputs.  Tolerances (BASELINE.json north_star):
max|ΔX|/max|X| <= 1e-10 for complex128, <= 2e-5 for complex64; the
reference's own fast-vs-naive bound 1e-12 (ref/tests/test_fastpath.py:146-154)
is used where the case comes from that test.
"""

import re

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 2e-5


@pytest.fixture(scope="module")
def asx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2403_16665_b200 as asx

    return asx


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def gpu_run(asx, x, a, d, m, method, dtype="complex128", real=False):
    """alpha_b = a/d on the GPU; x host (B, N) -> host (B, m)."""
    import torch

    alpha = asx.DenseFactor(d, a)
    p = asx.plan(x.shape[-1], alpha, m=m, dtype=dtype, method=method, real_input=real)
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    out = p.execute(xt)
    torch.cuda.synchronize()
    return out.cpu().numpy(), p


# ------------------------------------------------------------- known answers

def test_kat_two_sample_direct(asx, golden_kat):
    s = asx.naive_forward(asx.Signal([0.0, 1.0]), asx.DenseFactor(2))
    assert s.m == 4
    np.testing.assert_allclose(s.bins, golden_kat["two_sample_X"], atol=1e-15)


def test_kat_halving_direct(asx, golden_kat):
    s = asx.naive_forward(asx.Signal(golden_kat["halving_x"]), asx.DenseFactor(1, 2))
    np.testing.assert_allclose(s.bins, golden_kat["halving_X"], atol=1e-14)


@pytest.mark.parametrize("method", ["fft", "chirp", "direct"])
def test_kat_impulse(asx, golden_kat, method):
    p = asx.plan(4, asx.DenseFactor(2), method=method)
    s = asx.alpha_fft(asx.Signal([1.0, 0.0, 0.0, 0.0]), p)
    np.testing.assert_allclose(s.bins, golden_kat["impulse_X"], atol=1e-15)


def test_kat_combine_and_block_sum(asx, golden_kat):
    out = asx.combine(np.array([1.0 + 0j]), np.array([1.0 + 0j]), np.array([1.0 + 0j]))
    np.testing.assert_array_equal(out, golden_kat["combine_id"])
    out = asx.combine(np.array([0j]), np.array([1.0 + 0j]), np.array([-1j]))
    np.testing.assert_array_equal(out, golden_kat["combine_quarter"])
    out = asx.combine(golden_kat["combine_rows_y"], golden_kat["combine_rows_z"], golden_kat["combine_rows_tw"])
    np.testing.assert_allclose(out, golden_kat["combine_rows_out"], atol=1e-15)
    counter = asx.OpCounter()
    v = asx.leaf_block_sum(golden_kat["block_x"], counter)
    assert abs(v - golden_kat["block_sum"][0]) < 1e-14 and counter.complex_adds == 7
    with pytest.raises(ValueError):
        asx.combine(np.ones(2), np.ones(3), np.ones(2))


def test_plan_surface(asx, golden_kat, golden_counts):
    p = asx.plan(16, asx.DenseFactor(4))
    assert p.depth == 4 and p.shape == (64, 16) and p.leaf is asx.LeafKind.SINGLE_SAMPLE
    for k, t in enumerate(p.twiddles):
        np.testing.assert_allclose(t, golden_kat[f"twiddle_16_4_{k}"], atol=2e-16)
        with pytest.raises(ValueError):
            t[0] = 0
    for row in golden_counts:
        pl = asx.plan(row["n"], asx.DenseFactor(row["p"], row["q"]))
        assert (pl.m, pl.depth, pl.leaf.value) == (row["m"], row["depth"], row["leaf"])
        assert asx.predicted_mults(pl) == row["mults"] and asx.predicted_adds(pl) == row["adds"]
    with pytest.raises(asx.UnsupportedSizeError):
        asx.plan(12, asx.DenseFactor(1))
    with pytest.raises(asx.UnsupportedSizeError):
        asx.plan(8, asx.DenseFactor(3, 2))
    with pytest.raises(asx.IncompatibleAlphaError):
        asx.plan(4, asx.DenseFactor(3, 8))


def test_dft_matrix(asx, golden_kat):
    W = asx.dft_matrix(12, asx.DenseFactor(2, 3))
    np.testing.assert_allclose(W, golden_kat["dft_matrix_12_2_3"], atol=1e-15)
    W = asx.dft_matrix(256, asx.DenseFactor(100, 37), m=256, dtype="complex64")
    np.testing.assert_allclose(W, orc.dft_matrix(256, 37, 100, 256), atol=2e-7)


# ------------------------------------------------------------- golden grids

@pytest.mark.parametrize("method", ["fft", "chirp", "direct"])
def test_golden_fft_grid(asx, golden_grid_fft, method):
    worst = 0.0
    for key in golden_grid_fft:
        if not key.endswith("_x"):
            continue
        base = key[:-2]
        n, p, q = map(int, re.match(r"n(\d+)_p(\d+)_q(\d+)", base).groups())
        x = golden_grid_fft[key]
        want = golden_grid_fft[base + "_fft"]
        try:
            pl = asx.plan(n, asx.DenseFactor(p, q), method=method)
        except asx.UnsupportedSizeError:
            assert method == "chirp" and n * max(p, 1) // q + n > 8192
            continue
        got = asx.transform_samples(x, pl)
        assert got.shape == want.shape
        worst = max(worst, orc.rel_err(got, want))
    assert worst <= 1e-12, worst


def test_golden_naive_grid(asx, golden_grid_naive):
    worst = 0.0
    for key in golden_grid_naive:
        if not key.endswith("_x"):
            continue
        base = key[:-2]
        n, p, q = map(int, re.match(r"n(\d+)_p(\d+)_q(\d+)", base).groups())
        s = asx.naive_forward(asx.Signal(golden_grid_naive[key]), asx.DenseFactor(p, q))
        worst = max(worst, orc.rel_err(s.bins, golden_grid_naive[base + "_naive"]))
        for method in ("chirp", "direct"):
            pl = asx.plan(n, asx.DenseFactor(p, q), method=method)
            worst = max(worst, orc.rel_err(asx.transform_samples(golden_grid_naive[key], pl),
                                           golden_grid_naive[base + "_naive"]))
    assert worst <= 1e-12, worst


@pytest.mark.parametrize("method", ["direct", "fft", "chirp"])
def test_config0_golden(asx, golden_configs, method):
    x = golden_configs["c0_x"]
    for real in (True, False):
        xx = x if real else x.astype(np.complex128)
        got, p = gpu_run(asx, xx[None], 1, 4, 1024, method, real=real)
        assert orc.rel_err(got, golden_configs["c0_naive"][None]) <= TOL64
        assert orc.rel_err(got, golden_configs["c0_fft"][None]) <= TOL64


@pytest.mark.parametrize("method", ["direct", "fft", "chirp"])
def test_config_minis_golden(asx, golden_configs, method):
    got, _ = gpu_run(asx, golden_configs["c1b_mini_x"], 1, 10, 64, method)
    assert orc.rel_err(got, golden_configs["c1b_mini_X"]) <= TOL64
    got, _ = gpu_run(asx, golden_configs["c1a_mini_x"], 1, 2, 512, method)
    assert orc.rel_err(got, golden_configs["c1a_mini_X"]) <= TOL64
    got, _ = gpu_run(asx, golden_configs["c4_mini_x"], 1, 8, 256, method, dtype="complex64")
    assert orc.rel_err(got, golden_configs["c4_mini_X"]) <= TOL32


# ------------------------------------------------------- randomized vs oracle

CASES = [
    # (n, a, d, m, methods)
    (1, 1, 1, 1, ("fft", "chirp", "direct")),
    (2, 1, 3, 2, ("fft", "chirp", "direct")),
    (8, 1, 8, 8, ("fft", "chirp", "direct")),
    (64, 1, 5, 64, ("fft", "chirp", "direct")),
    (256, 37, 100, 256, ("chirp", "direct")),
    (256, 1, 8, 256, ("fft", "chirp", "direct")),
    (100, 3, 7, 77, ("chirp", "direct")),
    (1000, 1, 4, 1000, ("chirp", "direct")),
    (1024, 1, 2, 1024, ("fft", "chirp", "direct")),
    (1024, 4, 1, 256, ("fft", "chirp", "direct")),  # BLOCK_SUM leaf, alpha_ref 1/4
    (2048, 1, 10, 2048, ("fft", "chirp")),
    (4096, 1, 2, 4096, ("fft", "chirp")),
    (4096, 1, 10, 4096, ("fft", "chirp")),
    (8192, 1, 8, 8192, ("fft", "chirp")),
    (8192, 1, 1, 8192, ("fft", "chirp")),
    (512, 1, 4, 3000, ("fft", "chirp", "direct")),  # m > N, wraps past nothing (m < rN)
    (16, 1, 2, 80, ("fft", "direct")),  # m > r*N: periodic wrap
]


@pytest.mark.parametrize("n,a,d,m,methods", CASES)
@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_random_vs_oracle(asx, n, a, d, m, methods, dtype):
    rng = np.random.default_rng(n * 31 + a * 7 + d)
    batch = 3 if n >= 4096 else 5
    x = np.stack([orc.unit_disk(rng, n) for _ in range(batch)])
    if dtype == "complex64":
        x = x.astype(np.complex64)
    want = orc.direct(x.astype(np.complex128), a, d, m)
    tol = TOL64 if dtype == "complex128" else TOL32
    for method in methods:
        if dtype == "complex128" and method == "chirp" and 2 * n > 8192:
            continue  # complex128 chirp needs N+M-1 <= 8192
        got, p = gpu_run(asx, x, a, d, m, method, dtype=dtype)
        assert p.method == method
        err = orc.rel_err(got, want)
        assert err <= tol, (method, err)


def test_oversize_chirp_goes_four_step(asx):
    p = asx.plan(8192, asx.DenseFactor(8), m=8192, method="chirp", dtype="complex128")
    assert p.info.kernels_per_execute == 3 and p.fft_size == 16384
    with pytest.raises(asx.UnsupportedSizeError):
        asx.plan(1 << 23, asx.DenseFactor(8), m=1 << 23, method="chirp", dtype="complex128")


def test_alpha_fft_matches_reference_recursion_output(asx):
    # the GPU α-FFT vs the restated reference recursion, bins past N included
    rng = np.random.default_rng(12)
    x = np.stack([orc.unit_disk(rng, 512) for _ in range(4)])
    want = orc.alpha_fft(x, 1, 4)
    got, p = gpu_run(asx, x, 1, 4, None, "fft")
    assert p.m == 2048 and orc.rel_err(got, want) <= 1e-12


# --------------------------------------------------------------- edge cases

def test_empty_batch_and_strided_rows(asx, torch):
    p = asx.plan(64, asx.DenseFactor(4), m=64, method="fft")
    out = p.execute(torch.empty((0, 64), dtype=torch.complex128, device="cuda"))
    assert out.shape == (0, 64)
    rng = np.random.default_rng(4)
    big = torch.from_numpy(np.stack([orc.unit_disk(rng, 100) for _ in range(6)])).cuda()
    view = big[:, 10:74]  # row stride 100, inner stride 1
    for method in ("fft", "chirp", "direct"):
        pl = asx.plan(64, asx.DenseFactor(4), m=64, method=method)
        got = pl.execute(view).cpu().numpy()
        want = orc.direct(view.cpu().numpy(), 1, 4, 64)
        assert orc.rel_err(got, want) <= TOL64
        out = torch.zeros((6, 80), dtype=torch.complex128, device="cuda")
        with pytest.raises(ValueError):
            pl.execute(view, out=out)


def test_real_input_and_host_path(asx):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((7, 1024))
    want = orc.direct(x, 1, 4, 1024)
    for method in ("fft", "chirp", "direct"):
        pl = asx.plan(1024, asx.DenseFactor(4), m=1024, method=method, real_input=True)
        got = pl.execute_host(x, chunk=3)  # 3 chunks through the host pipeline
        assert orc.rel_err(got, want) <= TOL64


def test_wrong_length_raises(asx):
    p = asx.plan(8, asx.DenseFactor(2))
    with pytest.raises(ValueError):
        asx.alpha_fft(asx.Signal(np.ones(4)), p)
    with pytest.raises(ValueError):
        asx.transform_samples(np.ones(4, dtype=complex), p)


def test_counter_closed_forms(asx):
    p = asx.plan(8, asx.DenseFactor(2))
    c = asx.OpCounter()
    asx.alpha_fft(asx.Signal(np.ones(8)), p, c)
    assert c.complex_mults == 24 == asx.predicted_mults(p)
    c.reset()
    asx.transform_samples(np.ones((3, 8)), p, c)
    assert c.complex_mults == 72


def test_determinism(asx, torch):
    rng = np.random.default_rng(41)
    x = torch.from_numpy(np.stack([orc.unit_disk(rng, 4096) for _ in range(64)])).cuda()
    for method in ("fft", "chirp"):
        p = asx.plan(4096, asx.DenseFactor(2), m=4096, method=method)
        a = p.execute(x)
        b = p.execute(x)
        assert torch.equal(a, b)


def test_linearity_at_scale(asx, torch):
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((512, 8192), dtype=torch.complex64, device="cuda", generator=g)
    y = torch.randn((512, 8192), dtype=torch.complex64, device="cuda", generator=g)
    for method in ("fft", "chirp"):
        p = asx.plan(8192, asx.DenseFactor(8), m=8192, dtype="complex64", method=method)
        lhs = p.execute(x + 2 * y)
        rhs = p.execute(x) + 2 * p.execute(y)
        scale = lhs.abs().amax(dim=1)
        assert float(((lhs - rhs).abs().amax(dim=1) / scale).max()) <= TOL32


# ------------------------------------------------- four-step (large P) path

@pytest.mark.parametrize("n,a,d,m,dtype", [
    (8192, 1, 8, 8192, "complex128"),    # P = 16384 = 2 x 8192
    (6000, 3, 7, 5000, "complex128"),    # non-power-of-two N, non-dyadic alpha
    (16384, 1, 2, 16384, "complex64"),   # P = 32768 = 2 x 16384
    (1 << 18, 1, 16, 1 << 18, "complex64"),  # P = 2^19 = 32 x 16384
])
def test_large_chirp_vs_oracle(asx, n, a, d, m, dtype):
    rng = np.random.default_rng(n + d)
    x = np.stack([orc.unit_disk(rng, n) for _ in range(2)])
    if dtype == "complex64":
        x = x.astype(np.complex64)
    got, p = gpu_run(asx, x, a, d, m, "chirp", dtype=dtype)
    assert p.info.kernels_per_execute == 3 and p.fft_size > (8192 if dtype == "complex128" else 16384)
    if n * m <= (1 << 26):
        want = orc.direct(x.astype(np.complex128), a, d, m)
    else:  # zero-padded FFT == first M bins of the density-d spectrum (alpha = 1/d)
        assert a == 1
        want = np.fft.fft(x.astype(np.complex128), d * n, axis=1)[:, :m]
    tol = TOL64 if dtype == "complex128" else TOL32
    assert orc.rel_err(got, want) <= tol


@pytest.mark.parametrize("method", ["auto", "fft"])
def test_config2_full_size(asx, method):
    """BASELINE config 2: N = 2^22 real f64, alpha = 1/16, M = N: the four-step
    chirp (auto) and the paper's α-FFT recursion past one CTA (fft: 16 residues,
    each a four-step 2^22-point transform)."""
    from paper_2403_16665_b200.signals import WORKLOADS, generate

    w = WORKLOADS["2"]
    x = generate(w, 0, 1)[0]
    got, p = gpu_run(asx, x[None], 1, 16, w.m, method, real=True)
    assert p.method == ("chirp" if method == "auto" else "fft")
    if method == "fft":
        assert p.info.kernels_per_execute == 32
    # independent check: zero-padded FFT (pocketfft) of length 16N, first N bins
    want = np.fft.fft(x, 16 * w.n)[: w.m]
    assert orc.rel_err(got, want[None]) <= TOL64
    # the four-step twiddles are base x step powers of exact lookups (tw_chain_apply): measured 3e-16 on both
    # methods, pinned two orders above that so a lost exact seed shows up long before the 1e-10 bound
    assert orc.rel_err(got, want[None]) <= 5e-14
    # exact-reduction direct sums on sampled bins (ref/oracle.py:37-47 semantics)
    bins = np.array([0, 1, 7, 12345, w.m // 2, w.m - 1])
    nn = np.arange(w.n, dtype=np.int64)
    L = 16 * w.n
    for b in bins:
        idx = (b * nn) % L
        want_b = np.sum(x * np.exp(-2j * np.pi * idx / L))
        assert abs(got[0, b] - want_b) <= TOL64 * np.max(np.abs(got))


@pytest.mark.parametrize("n,d,m,real", [
    (16384, 2, 16384, False),        # P1 = 2
    (32768, 4, 20000, True),         # ragged M, real input
    (1 << 17, 8, 1 << 20, False),    # every bin of the density-8 spectrum (M = r N)
])
def test_large_alpha_fft_vs_oracle(asx, n, d, m, real):
    """The α-FFT past one CTA (four-step, one residue per launch pair) against
    the zero-padded FFT (first M bins of the density-d spectrum) and the oracle's
    exact-reduction sums on sampled bins."""
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((2, n)) if real else np.stack([orc.unit_disk(rng, n) for _ in range(2)])
    got, p = gpu_run(asx, x, 1, d, m, "fft", real=real)
    assert p.method == "fft" and p.info.kernels_per_execute == 2 * d
    want = np.fft.fft(x.astype(np.complex128), d * n, axis=1)[:, :m]
    assert orc.rel_err(got, want) <= TOL64
    # exact-reduction direct sums on sampled bins (ref/oracle.py:37-47 semantics)
    nn = np.arange(n, dtype=np.int64)
    for b in (0, 1, 5, m // 3, m - 1):
        want_b = (x * np.exp(-2j * np.pi * ((b * nn) % (d * n)) / (d * n))).sum(axis=1)
        assert np.max(np.abs(got[:, b] - want_b)) <= TOL64 * np.max(np.abs(got))
    # the reference's plan() rule past one CTA: power-of-two density only
    with pytest.raises(asx.UnsupportedSizeError):
        asx.plan(16384, asx.DenseFactor(3), m=16384, method="fft")
    with pytest.raises(asx.UnsupportedSizeError):
        asx.plan(16384, asx.DenseFactor(2), m=16384, dtype="complex64", method="fft")


def test_lazy_conjugate_views_are_resolved(asx, torch):
    rng = np.random.default_rng(8)
    x = torch.from_numpy(np.stack([orc.unit_disk(rng, 64) for _ in range(3)])).cuda()
    p = asx.plan(64, asx.DenseFactor(2), m=64)
    got = p.execute(x.conj()).cpu().numpy()
    want = orc.direct(np.conj(x.cpu().numpy()), 1, 2, 64)
    assert orc.rel_err(got, want) <= TOL64


def test_four_step_reentrant_across_streams(asx, torch):
    """The four-step path keeps one workspace per stream: concurrent executes on
    two streams and the host path's stream ring give the single-stream result."""
    rng = np.random.default_rng(77)
    x = np.stack([orc.unit_disk(rng, 8192) for _ in range(6)])
    p = asx.plan(8192, asx.DenseFactor(8), m=8192, method="chirp", dtype="complex128")
    assert p.info.kernels_per_execute == 3
    xt = torch.from_numpy(x).cuda()
    want = p.execute(xt)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for s, rows in ((s1, slice(0, 3)), (s2, slice(3, 6))):
        with torch.cuda.stream(s):
            outs.append(p.execute(xt[rows]))
    torch.cuda.synchronize()
    got = torch.cat(outs)
    assert torch.equal(got, want)
    host = p.execute_host(x, chunk=1)  # six chunks over the three-stream ring
    np.testing.assert_array_equal(host, want.cpu().numpy())


def test_complex64_fft_is_fp64_inside(asx, torch):
    # the α-FFT recursion of a complex64 plan runs in FP64: its
    # error is the complex64 output rounding only, far below the bound even on
    # signals whose energy lies outside the M-bin window (config 4's hard case)
    n = 8192
    t = np.arange(n)
    rng = np.random.default_rng(77)
    rows = []
    for _ in range(4):  # tones at f > N/8: none falls inside the alpha = 1/8 window
        f = rng.uniform(n / 8 + 50, n / 2 - 50, 4)
        ph = rng.uniform(0, 2 * np.pi, 4)
        sig = sum(np.exp(2j * np.pi * fk * t / n + 1j * pk) for fk, pk in zip(f, ph))
        rows.append(sig + 0.1 * (rng.standard_normal(n) + 1j * rng.standard_normal(n)))
    x = np.stack(rows).astype(np.complex64)
    want = orc.direct(x.astype(np.complex128), 1, 8, n)
    got, p = gpu_run(asx, x, 1, 8, n, "fft", dtype="complex64")
    assert p.method == "fft"
    assert orc.rel_err(got, want) <= 1e-6
    # the FP64 engine's inner size limit applies to complex64 plans too
    with pytest.raises(asx.UnsupportedSizeError):
        asx.plan(16384, asx.DenseFactor(1), m=16384, dtype="complex64", method="fft")


def test_leading_dims_flatten_into_the_batch(asx, torch):
    rng = np.random.default_rng(9)
    x = np.stack([orc.unit_disk(rng, 256) for _ in range(6)]).reshape(2, 3, 256)
    want = orc.direct(x.reshape(6, 256), 1, 2, 256).reshape(2, 3, 256)
    p = asx.plan(256, asx.DenseFactor(2), m=256, method="fft")
    got = p.execute(torch.from_numpy(x).cuda())
    assert tuple(got.shape) == (2, 3, 256)
    assert orc.rel_err(got.cpu().numpy().reshape(6, 256), want.reshape(6, 256)) <= TOL64
    got_h = p.execute_host(x)
    assert got_h.shape == (2, 3, 256)
    assert orc.rel_err(got_h.reshape(6, 256), want.reshape(6, 256)) <= TOL64


def test_four_step_batched_groups(asx, torch):
    """The four-step path transforms the batch in groups of batch_group
    signals per launch set (workspace group x P): complex128 N = 8192,
    alpha = 1/8 (config 4's shape at FP64), 4096 signals = 2 groups of 2048,
    every signal against the single-CTA alpha-FFT recursion; plus a batched
    large alpha-FFT against the zero-padded FFT."""
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn((4096, 8192), dtype=torch.complex128, device="cuda", generator=g)
    p = asx.plan(8192, asx.DenseFactor(8), m=8192, dtype="complex128", method="chirp")
    assert p.info.kernels_per_execute == 3 and p.info.batch_group == 2048
    q = asx.plan(8192, asx.DenseFactor(8), m=8192, dtype="complex128", method="fft")
    got, want = p.execute(x), q.execute(x)
    err = ((got - want).abs().amax(dim=1) / want.abs().amax(dim=1)).max().item()
    assert err <= 2 * TOL64, err
    # ragged batch across the group boundary, strided rows
    sub = x[5:2060]
    assert torch.equal(p.execute(sub), got[5:2060])
    rng = np.random.default_rng(3)
    xs = np.stack([orc.unit_disk(rng, 16384) for _ in range(5)])
    got2, p2 = gpu_run(asx, xs, 1, 2, 16384, "fft")
    assert p2.info.batch_group >= 5
    assert orc.rel_err(got2, np.fft.fft(xs, 2 * 16384, axis=1)[:, :16384]) <= TOL64
