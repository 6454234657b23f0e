"""The bench grid's schema and claims against the REFERENCE's own report
(tests/golden/gridbench_ref.{json,csv}, made by make_gridbench_golden.py
from ref/bench.py:210-422): same runnable cells in the same order, the same
skip reasons, exact operation counts, identical verdicts for the same
records, identical JSON / CSV layout.  No GPU needed: only the timing in
run_grid touches the device (tests/test_gpu_gridbench.py)."""

import csv
import io
import json
import os

import pytest

from paper_2403_16665_b200 import DenseFactor
from paper_2403_16665_b200 import gridbench as gb

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "gridbench_ref.json")) as fh:
        return json.load(fh)


def _records(rows):
    return [gb.BenchRecord(r["N"], DenseFactor(r["alpha_p"], r["alpha_q"]), r["method"], r["mults"], r["adds"],
                           r["wall_ns"] / 1e9, r["reps"]) for r in rows]


def test_cells_and_skips_match_reference(golden):
    g = golden["grid"]
    skipped = []
    cells = gb.grid_cells(g["ns"], [DenseFactor(p, q) for p, q in g["alphas"]], g["methods"], skipped)
    rows = golden["report"]["records"]
    assert [(n, (a.p, a.q), m) for n, a, m in cells] == [(r["N"], (r["alpha_p"], r["alpha_q"]), r["method"])
                                                         for r in rows]
    assert skipped == golden["report"]["skipped"]


def test_counts_are_the_reference_counters(golden):
    for r in golden["report"]["records"]:
        assert gb.cell_counts(r["N"], DenseFactor(r["alpha_p"], r["alpha_q"]), r["method"]) == (r["mults"], r["adds"])


def test_report_equals_reference_report(golden):
    recs = _records(golden["report"]["records"])
    rep = gb.make_report(recs, golden["report"]["skipped"])
    got = json.loads(json.dumps(rep.to_dict()))
    want = golden["report"]
    assert got["records"] == want["records"]
    assert got["skipped"] == want["skipped"]
    assert len(got["verdicts"]) == len(want["verdicts"])
    for a, b in zip(got["verdicts"], want["verdicts"]):
        assert (a["claim"], a["pass"], a["record_ids"], a["warnings"]) == (b["claim"], b["pass"], b["record_ids"],
                                                                          b["warnings"])
        assert len(a["details"]) == len(b["details"])
        for da, db in zip(a["details"], b["details"]):
            assert da.keys() == db.keys()
            for k in da:
                assert da[k] == pytest.approx(db[k], rel=1e-12) if isinstance(db[k], float) else da[k] == db[k]
    assert rep.all_passed


def test_csv_layout(golden, tmp_path):
    recs = _records(golden["report"]["records"])
    path = tmp_path / "r.csv"
    gb.ScalingReport(recs, []).write_csv(path)
    with open(os.path.join(GOLDEN, "gridbench_ref.csv")) as fh:
        assert path.read_text() == fh.read()


def test_record_validation_and_failed_claim():
    good = gb.BenchRecord(8, DenseFactor(2), "alpha_fft", 24, 48, 1e-6, 3)
    assert good.to_row() == {"N": 8, "alpha_p": 2, "alpha_q": 1, "method": "alpha_fft", "mults": 24, "adds": 48,
                             "wall_ns": 1000, "reps": 3}
    for bad in [("butterfly", 24, 1e-6, 3), ("alpha_fft", -1, 1e-6, 3), ("alpha_fft", 24, 0.0, 3),
                ("alpha_fft", 24, 1e-6, 0)]:
        with pytest.raises(ValueError):
            gb.BenchRecord(8, DenseFactor(2), bad[0], bad[1], 48, bad[2], bad[3])
    # a zeropad count that does not exceed the α-FFT count by (αN/2) log2 α fails the claim
    recs = [gb.BenchRecord(256, DenseFactor(2), "alpha_fft", 2048, 4096, 1e-6, 1),
            gb.BenchRecord(256, DenseFactor(2), "zeropad_fft", 2049, 4608, 1e-6, 1)]
    v = gb.check_alpha_gt1_savings(recs)
    assert not v.passed and v.details[0]["expected_gap"] == 256
    with pytest.raises(gb.IncompleteGridError):
        gb.check_alpha_lt1_savings(recs)
    with pytest.raises(gb.IncompleteGridError):
        gb.fit_complexity(recs)
    assert gb.cell_validity(8, DenseFactor(1, 3), "naive") == (False, "alpha*N = 8/3 is not an integer")
