"""`bench` on GPU plans end to end (ref tests/test_cli.py:132-168 and
test_bench.py as the model): device-timed records in the reference's JSON /
CSV schema, all scaling claims passing, skip and exit-code behaviour."""

import csv
import json

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cli():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2403_16665_b200 import cli

    return cli


def test_bench_writes_reports_and_passes(cli, tmp_path, capsys):
    jp, cp = tmp_path / "report.json", tmp_path / "records.csv"
    code = cli.main(["bench", "--grid-n", "64,128,256,512", "--grid-alpha", "1/2,1,2", "--reps", "2",
                     "--methods", "alpha_fft,zeropad_fft,naive", "--output", str(jp), "--csv", str(cp)])
    out = capsys.readouterr().out
    assert code == cli.EXIT_OK
    for claim in ("alpha_gt1_savings", "alpha_lt1_savings", "complexity_fit_alpha_2_1"):
        assert f"claim {claim}: pass" in out
    assert "skipped" in out  # alpha < 1 zeropad cells
    rep = json.loads(jp.read_text())
    assert set(rep) == {"records", "verdicts", "skipped"}
    assert all(set(r) == {"N", "alpha_p", "alpha_q", "method", "mults", "adds", "wall_ns", "reps"}
               for r in rep["records"])
    assert all(r["wall_ns"] > 0 for r in rep["records"])
    assert all(set(v) == {"claim", "pass", "record_ids", "details", "warnings"} for v in rep["verdicts"])
    with open(cp) as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == len(rep["records"])
    fast = [r for r in rep["records"] if (r["N"], r["alpha_p"], r["method"]) == (256, 2, "alpha_fft")][0]
    assert (fast["mults"], fast["adds"]) == (2048, 4096)  # ref test_bench.py:70-77


def test_bench_empty_grid(cli, capsys):
    assert cli.main(["bench", "--grid-n", "12", "--grid-alpha", "1", "--reps", "1"]) == cli.EXIT_PARSE_ERROR
    assert "no runnable grid cells" in capsys.readouterr().err


def test_bench_rejects_unknown_method(cli):
    with pytest.raises(SystemExit) as info:
        cli.main(["bench", "--methods", "fastest"])
    assert info.value.code == 2
