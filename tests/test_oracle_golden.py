"""Pin the CPU oracle (oracle/alpha_oracle.py) to the reference's own outputs.

The golden vectors were produced by the reference package itself
(tests/golden/make_golden.py); the known-answer cases mirror the reference's
tests (ref/tests/test_oracle.py:35-45, ref/tests/test_fastpath.py:102-143).
"""

import cmath
import re

import numpy as np
import pytest

from oracle import alpha_oracle as orc

TOL_C128 = 1e-12  # reference oracle-equivalence bound (ref/tests/test_fastpath.py:146-154)


def _cases(golden, suffix):
    for key in golden:
        if key.endswith("_x"):
            base = key[:-2]
            if base + suffix in golden:
                yield base, golden[key], golden[base + suffix]


def test_kat_two_sample(golden_kat):
    got = orc.direct(golden_kat["two_sample_x"], 1, 2, 4)[0]  # DenseFactor(2) = alpha_b 1/2
    np.testing.assert_allclose(got, golden_kat["two_sample_X"], atol=1e-15)
    np.testing.assert_allclose(got, [1, -1j, -1, 1j], atol=1e-15)


def test_kat_halving(golden_kat):
    x = golden_kat["halving_x"]
    got = orc.direct(x, 2, 1, 2)[0]  # DenseFactor(1, 2) = alpha_b 2
    np.testing.assert_allclose(got, golden_kat["halving_X"], atol=1e-14)
    a, b, c, d = x
    np.testing.assert_allclose(got, [a + b + c + d, a - b + c - d], atol=1e-14)


def test_kat_impulse(golden_kat):
    got = orc.alpha_fft(np.array([1.0, 0, 0, 0]), 1, 2)[0]
    np.testing.assert_array_equal(got, golden_kat["impulse_X"])
    np.testing.assert_array_equal(got, np.ones(8))


def test_kat_combine(golden_kat):
    np.testing.assert_array_equal(orc.combine(np.array([1 + 0j]), np.array([1 + 0j]), np.array([1 + 0j])),
                                  golden_kat["combine_id"])
    np.testing.assert_array_equal(orc.combine(np.array([0j]), np.array([1 + 0j]), np.array([-1j])),
                                  golden_kat["combine_quarter"])
    got = orc.combine(golden_kat["combine_rows_y"], golden_kat["combine_rows_z"], golden_kat["combine_rows_tw"])
    np.testing.assert_array_equal(got, golden_kat["combine_rows_out"])
    with pytest.raises(ValueError):
        orc.combine(np.ones(2), np.ones(3), np.ones(2))


def test_kat_block_sum(golden_kat):
    assert orc.leaf_block_sum(golden_kat["block_x"]) == golden_kat["block_sum"][0]


def test_twiddle_tables_bit_exact(golden_kat):
    tables = orc.plan_twiddles(64, 4)  # plan(16, DenseFactor(4)): m_ref 64, depth 4
    for k, t in enumerate(tables):
        np.testing.assert_array_equal(t, golden_kat[f"twiddle_16_4_{k}"])


def test_dft_matrix_non_dyadic(golden_kat):
    # DenseFactor(2, 3) at N=12 -> alpha_b = 3/2, 8 rows
    got = orc.dft_matrix(12, 3, 2, 8)
    np.testing.assert_allclose(got, golden_kat["dft_matrix_12_2_3"], atol=1e-15)


def test_alpha_fft_matches_reference_fast_path(golden_grid_fft):
    worst = 0.0
    count = 0
    for key, x, want in _cases(golden_grid_fft, "_fft"):
        n, p, q = map(int, re.match(r"n(\d+)_p(\d+)_q(\d+)", key).groups())
        got = orc.alpha_fft(x, q, p)[0]  # alpha_b = q/p
        # same recursion, same tables: bit-identical to the reference
        np.testing.assert_array_equal(got, want, err_msg=key)
        worst = max(worst, orc.rel_err(got, want))
        count += 1
    assert count > 100 and worst == 0.0


def test_direct_matches_reference_naive(golden_grid_fft, golden_grid_naive):
    worst = 0.0
    for golden in (golden_grid_fft, golden_grid_naive):
        for key, x, want in _cases(golden, "_naive"):
            n, p, q = map(int, re.match(r"n(\d+)_p(\d+)_q(\d+)", key).groups())
            got = orc.direct(x, q, p, want.size)[0]
            worst = max(worst, orc.rel_err(got, want))
    assert worst < TOL_C128


def test_restatement_matches_scalar_definition():
    # from-scratch scalar loop of the BASELINE formula, incl. alpha the reference rejects
    rng = np.random.default_rng(5)
    for (n, a, d, m) in [(8, 37, 100, 8), (6, 3, 2, 5), (5, 1, 3, 7), (12, 2, 3, 12)]:
        x = orc.unit_disk(rng, n)
        want = np.array([sum(x[j] * cmath.exp(-2j * cmath.pi * ((a * k * j) % (d * n)) / (d * n))
                             for j in range(n)) for k in range(m)])
        got = orc.direct(x, a, d, m)[0]
        assert orc.rel_err(got, want) < 1e-13


def test_oracle_on_config0_fixture(golden_configs):
    x = golden_configs["c0_x"]
    assert orc.rel_err(orc.direct(x, 1, 4, 1024), golden_configs["c0_naive"]) < 1e-13
    np.testing.assert_array_equal(orc.alpha_fft(x, 1, 4, 1024)[0], golden_configs["c0_fft"])


def test_oracle_on_config_minis(golden_configs):
    assert orc.rel_err(orc.direct(golden_configs["c1b_mini_x"], 1, 10, 64), golden_configs["c1b_mini_X"]) < 1e-13
    # non-power-of-two density r=10 through the generalised recursion
    assert orc.rel_err(orc.alpha_fft(golden_configs["c1b_mini_x"], 1, 10, 64), golden_configs["c1b_mini_X"]) < 1e-13
    x4 = golden_configs["c4_mini_x"].astype(np.complex128)
    np.testing.assert_array_equal(orc.alpha_fft(x4, 1, 8, 256), golden_configs["c4_mini_X"])
    np.testing.assert_array_equal(orc.alpha_fft(golden_configs["c1a_mini_x"], 1, 2, 512), golden_configs["c1a_mini_X"])


def test_predicted_counts(golden_counts):
    for row in golden_counts:
        assert orc.predicted_mults(row["n"], row["m"]) == row["mults"]
        assert orc.predicted_adds(row["n"], row["m"]) == row["adds"]


def test_rel_err_metric():
    want = np.array([[1.0, 2.0], [4.0, 0.0]])
    got = want + np.array([[0.2, 0.0], [0.0, 0.4]])
    assert orc.rel_err(got, want) == pytest.approx(0.1)
