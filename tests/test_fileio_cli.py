"""File formats and CLI argument handling (host side, no GPU) — mirrors
ref/tests/test_io.py and the parse-error / exit-code paths of ref/tests/test_cli.py."""

import json

import numpy as np
import pytest

from paper_2403_16665_b200 import DenseFactor, Signal, Spectrum, cli, fileio


def test_signal_csv_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    sig = Signal(rng.standard_normal(9) + 1j * rng.standard_normal(9), duration=0.25)
    path = tmp_path / "s.csv"
    fileio.write_signal_csv(sig, path)
    back = fileio.read_signal(path)
    assert back.duration == 0.25 and np.array_equal(back.samples, sig.samples)
    text = path.read_text()
    fileio.write_signal_csv(back, path)
    assert path.read_text() == text  # 17 significant digits: byte-exact


def test_time_value_csv_and_json(tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("time,value\n0,1\n0.5,2\n1.0,3\n")
    s = fileio.read_signal(p)
    assert s.duration == pytest.approx(1.5) and np.array_equal(s.samples, [1, 2, 3])
    j = tmp_path / "s.json"
    j.write_text(json.dumps({"T": 2.0, "samples": [1, [0, 1], 2.5]}))
    s = fileio.read_signal(j)
    assert s.duration == 2.0 and np.array_equal(s.samples, [1, 1j, 2.5])
    j.write_text(json.dumps({"time": [0, 1, 2], "value": [4, 5, 6]}))
    assert fileio.read_signal(j).duration == pytest.approx(3.0)


@pytest.mark.parametrize("body, fragment", [
    ("index,re,im\n1,0,0\n", "out of order"),
    ("foo,bar\n1,2\n", "expected header"),
    ("index,re,im\n0,x,0\n", "expected a number"),
    ("time,value\n0,1\n1,2\n3,3\n", "uniformly"),
    ("# N=3\nindex,re,im\n0,1,0\n", "declares N=3"),
])
def test_signal_parse_errors(tmp_path, body, fragment):
    p = tmp_path / "bad.csv"
    p.write_text(body)
    with pytest.raises(fileio.SignalParseError, match=fragment):
        fileio.read_signal(p)


def test_spectrum_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    spec = Spectrum(rng.standard_normal(8) + 1j * rng.standard_normal(8), 4, DenseFactor(2), 1.5)
    path = tmp_path / "x.csv"
    fileio.write_spectrum(spec, path, "fft")
    back, method = fileio.read_spectrum(path)
    assert method == "fft" and back.alpha == DenseFactor(2) and np.array_equal(back.bins, spec.bins)
    partial = Spectrum(spec.bins[:3], 4, DenseFactor(2), 1.5, m_bins=3)
    fileio.write_spectrum(partial, path, "chirp")
    back, _ = fileio.read_spectrum(path)
    assert back.m == 3


def test_cli_parse_errors_exit_codes(tmp_path, capsys):
    assert cli.main(["compute", "--input", str(tmp_path / "missing.csv"), "--output", str(tmp_path / "o.csv")]) == 2
    bad = tmp_path / "bad.csv"
    bad.write_text("nope\n")
    assert cli.main(["compute", "--input", str(bad), "--output", str(tmp_path / "o.csv")]) == 2
    with pytest.raises(SystemExit):
        cli.main(["compute", "--input", "a", "--output", "b", "--alpha", "1.5"])
