"""Host-side logic of the drop-in API: domain types, α conventions, workloads."""

from fractions import Fraction

import numpy as np
import pytest

from paper_2403_16665_b200 import (
    DenseFactor,
    IncompatibleAlphaError,
    Signal,
    Spectrum,
    density_for_alpha,
    validate_pair,
)
from paper_2403_16665_b200.signals import WORKLOADS, generate


def test_dense_factor_reduces_and_rejects():
    assert DenseFactor(4, 2) == DenseFactor(2, 1)
    with pytest.raises(ValueError):
        DenseFactor(0, 1)
    with pytest.raises(ValueError):
        DenseFactor(1.5, 1)
    assert DenseFactor.from_string("6/4") == DenseFactor(3, 2)
    with pytest.raises(ValueError):
        DenseFactor.from_string("1/2/3")


def test_validate_pair_rule():
    assert validate_pair(8, DenseFactor(3, 2)) == (8, 12)
    with pytest.raises(IncompatibleAlphaError) as exc:
        validate_pair(256, DenseFactor(100, 37))
    assert exc.value.n == 256 and exc.value.p == 100 and exc.value.q == 37


def test_baseline_alpha_convention():
    # alpha_b = 1/alpha_ref, taken exactly
    assert density_for_alpha("0.25") == DenseFactor(4)
    assert density_for_alpha("0.1") == DenseFactor(10)
    assert density_for_alpha("1/16") == DenseFactor(16)
    assert density_for_alpha("0.37") == DenseFactor(100, 37)
    assert DenseFactor(100, 37).alpha_b == Fraction(37, 100)
    with pytest.raises(ValueError):
        density_for_alpha(0.37)


def test_spectrum_explicit_bin_count():
    with pytest.raises(ValueError):
        Spectrum(np.zeros(4), 4, DenseFactor(2))
    s = Spectrum(np.zeros(4), 4, DenseFactor(2), m_bins=4)
    assert s.m == 4 and not s.bins.flags.writeable
    s = Spectrum(np.zeros(256), 256, DenseFactor(100, 37), m_bins=256)
    assert s.bin_frequency(1) == pytest.approx(0.37)


def test_signal_copies_to_readonly_c128():
    raw = np.arange(4, dtype=np.float32)
    s = Signal(raw)
    assert s.samples.dtype == np.complex128 and not s.samples.flags.writeable
    raw[0] = 7
    assert s.samples[0] == 0


def test_workload_algorithmic_figures():
    # SURVEY.md §8(d) table
    w = WORKLOADS["1a"]
    assert w.bytes_alg() == 536_870_912
    assert w.flops_alg(1) == 6 * 49_152 + 2 * 98_304
    assert WORKLOADS["1b"].flops_alg(1) == 6 * 245_760 + 2 * 491_520
    assert WORKLOADS["4"].bytes_alg() == 8_589_934_592
    assert WORKLOADS["4"].flops_alg(1) == 6 * 425_984 + 2 * 851_968
    assert WORKLOADS["3"].bytes_alg() == 1_073_741_824
    assert WORKLOADS["3"].flops_alg(1) == 8 * 256 * 256
    assert WORKLOADS["2"].flops_alg() == 6 * 738_197_504 + 2 * 1_476_395_008


def test_generator_is_per_signal_reproducible():
    w = WORKLOADS["4"]
    a = generate(w, 10, 3, threads=1)
    b = generate(w, 11, 1, threads=1)
    assert a.dtype == np.complex64 and a.shape == (3, 8192)
    np.testing.assert_array_equal(a[1], b[0])
    x0 = generate(WORKLOADS["0"], 0, 1)
    assert x0.dtype == np.float64 and x0.shape == (1, 1024)
