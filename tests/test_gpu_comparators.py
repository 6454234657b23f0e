"""GPU parity of SURVEY.md §8(f) rows 1-2: inverse α-DFT, orthogonality comb,
zero-pad comparator, alias fold — against the reference's golden vectors and
the reference tests' properties (ref/tests/test_oracle.py:117-160,
ref/tests/test_acceptance.py:79-110, ref/tests/test_baseline.py)."""

import re

import numpy as np
import pytest

from oracle import alpha_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def asx():
    import torch

    assert torch.cuda.is_available()
    import paper_2403_16665_b200 as asx

    return asx


def test_inverse_matches_reference(asx, golden_kat):
    cases = 0
    for key in golden_kat:
        m = re.match(r"inv_n(\d+)_p(\d+)_q(\d+)_X$", key)
        if not m:
            continue
        n, p, q = map(int, m.groups())
        spec = asx.Spectrum(golden_kat[key], n, asx.DenseFactor(p, q), duration=2.0)
        got = asx.naive_inverse(spec)
        want = golden_kat[key[:-2] + "_x"]
        assert got.duration == 2.0 and len(got) == n
        assert np.max(np.abs(got.samples - want)) < 1e-12
        cases += 1
    assert cases == 7


@pytest.mark.parametrize("n, p, q", [(8, 1, 1), (8, 2, 1), (16, 4, 1), (12, 3, 2), (64, 1, 1), (4096, 2, 1)])
def test_round_trip_recovers_signal(asx, n, p, q):
    rng = np.random.default_rng(1000 + n)
    sig = asx.Signal(orc.unit_disk(rng, n), duration=2.0)
    back = asx.naive_inverse(asx.alpha_fft(sig, asx.plan(n, asx.DenseFactor(p, q), method="auto")))
    assert np.max(np.abs(back.samples - sig.samples)) < 1e-10


@pytest.mark.parametrize("n, q", [(16, 2), (16, 4), (32, 8), (12, 3)])
def test_inverse_alias_sum(asx, golden_kat, n, q):
    rng = np.random.default_rng(n * q + 1)
    x = orc.unit_disk(rng, n)
    back = asx.naive_inverse(asx.naive_forward(asx.Signal(x), asx.DenseFactor(1, q))).samples
    folded = asx.aliased_reconstruct(asx.Signal(x), asx.DenseFactor(1, q))
    m = n // q
    want = np.array([x[s % m::m].sum() for s in range(n)])
    assert np.max(np.abs(back - want)) < 1e-12
    assert np.max(np.abs(folded - want)) < 1e-13
    for key in golden_kat:
        mm = re.match(r"alias_n(\d+)_p(\d+)_q(\d+)$", key)
        if mm:
            nn, pp, qq = map(int, mm.groups())
            got = asx.aliased_reconstruct(asx.Signal(golden_kat[key + "_in"]), asx.DenseFactor(pp, qq))
            assert np.max(np.abs(got - golden_kat[key])) < 1e-13


def test_orthogonality_comb(asx, golden_kat):
    got = np.array([asx.orthogonality_kernel(d, 0, 12, asx.DenseFactor(3, 2)) for d in range(-11, 12)])
    assert np.max(np.abs(got - golden_kat["orth_12_3_2"])) < 1e-12
    for d in range(-11, 12):
        v = asx.orthogonality_kernel(d, 0, 12, asx.DenseFactor(3, 2))
        if d % 18 == 0:
            assert v == 1.0
        else:
            assert abs(v) < 1e-12


def test_zero_pad_equivalence(asx, golden_kat):
    sig = asx.Signal(golden_kat["zeropad_x"])
    padded = asx.standard_fft(asx.zero_pad(sig, asx.DenseFactor(4)))
    assert np.max(np.abs(padded.bins - golden_kat["zeropad_X"])) < 1e-12
    dense = asx.alpha_fft(sig, asx.plan(32, asx.DenseFactor(4)))
    assert np.max(np.abs(dense.bins - padded.bins)) < 1e-12  # criterion 2 (ref test_acceptance.py:79-90)
    with pytest.raises(ValueError):
        asx.zero_pad(sig, asx.DenseFactor(1, 2))
    with pytest.raises(ValueError):
        asx.aliased_reconstruct(sig, asx.DenseFactor(2))


def test_standard_fft_is_numpy_fft(asx):
    rng = np.random.default_rng(77)
    x = orc.unit_disk(rng, 128)
    assert np.max(np.abs(asx.standard_fft(x).bins - np.fft.fft(x))) < 1e-11
    x = orc.unit_disk(rng, 100)  # non-power-of-two: chirp path
    assert np.max(np.abs(asx.standard_fft(x).bins - np.fft.fft(x))) < 1e-11


def test_cli_compute_and_verify(asx, tmp_path, golden_configs):
    from paper_2403_16665_b200 import cli, fileio

    sig = asx.Signal(golden_configs["c0_x"])
    src = tmp_path / "sig.csv"
    fileio.write_signal_csv(sig, src)
    for method in ("auto", "fft", "naive", "zeropad", "chirp"):
        out = tmp_path / f"spec_{method}.csv"
        assert cli.main(["compute", "--input", str(src), "--output", str(out), "--alpha", "4",
                         "--method", method]) == 0
        spec, used = fileio.read_spectrum(out)
        assert spec.m == 4096
        assert np.max(np.abs(spec.bins[:1024] - golden_configs["c0_naive"])) / np.max(
            np.abs(golden_configs["c0_naive"])) < 1e-10
    # explicit bin count (BASELINE's M = N) and an alpha the reference rejects
    out = tmp_path / "m.csv"
    assert cli.main(["compute", "--input", str(src), "--output", str(out), "--alpha", "100/37",
                     "--bins", "1024"]) == 0
    assert cli.main(["compute", "--input", str(src), "--output", str(out), "--alpha", "100/37"]) == 3
    assert cli.main(["compute", "--input", str(src), "--output", str(out), "--alpha", "3/2",
                     "--method", "fft"]) == 4
    assert cli.main(["verify", "--sizes", "2,4,8,16"]) == 0
    assert cli.main(["verify", "--sizes", "4", "--inject-fault"]) == 1


def test_gpu_verify_suites(asx):
    from paper_2403_16665_b200 import verify

    for r in verify.run_all(seed=0):
        assert r.passed, (r.name, r.max_error, r.worst)
