"""Signal / spectrum files of the reference CLI.

The formats are the reference's (ref/io.py:1-8): signal CSV with an
``index,re,im`` or ``time,value`` header and ``# key=value`` metadata lines
(``T``, ``N``), signal JSON (``{"samples": [...]}`` or ``{"time", "value"}``),
and spectrum CSV with ``# N / alpha / T / method`` metadata followed by
``m,freq,re,im,magnitude`` rows, floats printed with 17 significant digits so
files round-trip exactly.  Parsing is host-side text handling; the transform
itself runs on the GPU.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .core import DenseFactor, Signal, Spectrum, bin_frequency

UNIFORM_RTOL = 1e-9


class SignalParseError(ValueError):
    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


def fmt17(v: float) -> str:
    return format(float(v), ".17g")


def _num(text: str, line):
    try:
        return float(text)
    except ValueError:
        raise SignalParseError(f"expected a number, got {text!r}", line) from None


def _meta(body: str, line, out: dict) -> None:
    key, sep, val = body.partition("=")
    if not sep:
        return
    key, val = key.strip(), val.strip()
    if key == "T":
        out["T"] = _num(val, line)
    elif key == "N":
        try:
            out["N"] = int(val)
        except ValueError:
            raise SignalParseError(f"expected an integer N, got {val!r}", line) from None
    elif key == "alpha":
        try:
            out["alpha"] = DenseFactor.from_string(val)
        except ValueError as exc:
            raise SignalParseError(str(exc), line) from None
    elif key == "method":
        out["method"] = val


def _csv_rows(path):
    """Yield (line_no, cells) of data rows; metadata lines fill the returned dict."""
    meta, rows = {}, []
    for line_no, raw in enumerate(Path(path).read_text().splitlines(), start=1):
        s = raw.strip()
        if not s:
            continue
        if s.startswith("#"):
            _meta(s.lstrip("#").strip(), line_no, meta)
        else:
            rows.append((line_no, [c.strip() for c in s.split(",")]))
    return meta, rows


def _uniform_duration(times, line):
    steps = np.diff(np.asarray(times, dtype=float))
    if steps.size == 0:
        return None
    dt = float(steps.mean())
    if dt <= 0 or float(np.max(np.abs(steps - dt))) > UNIFORM_RTOL * abs(dt):
        raise SignalParseError("time values are not uniformly spaced", line)
    return dt * len(times)


def read_signal_csv(path) -> Signal:
    meta, rows = _csv_rows(path)
    if not rows:
        raise SignalParseError("no header row found")
    (hline, header), body = rows[0], rows[1:]
    kind = [c.lower() for c in header]
    if kind not in (["index", "re", "im"], ["time", "value"]):
        raise SignalParseError(f"expected header 'index,re,im' or 'time,value', got {','.join(header)!r}", hline)
    if not body:
        raise SignalParseError("no sample rows found")
    for line_no, cells in body:
        if len(cells) != len(kind):
            raise SignalParseError(f"expected {len(kind)} columns, got {len(cells)}", line_no)
    if kind[0] == "index":
        samples = np.empty(len(body), dtype=np.complex128)
        for pos, (line_no, (idx, re, im)) in enumerate(body):
            try:
                ii = int(idx)
            except ValueError:
                raise SignalParseError(f"expected an integer index, got {idx!r}", line_no) from None
            if ii != pos:
                raise SignalParseError(f"index {ii} out of order (expected {pos})", line_no)
            samples[pos] = complex(_num(re, line_no), _num(im, line_no))
        duration = meta.get("T", 1.0)
    else:
        times = [_num(c[0], ln) for ln, c in body]
        samples = np.array([_num(c[1], ln) for ln, c in body], dtype=np.complex128)
        derived = _uniform_duration(times, body[-1][0])
        duration = meta.get("T", derived if derived is not None else 1.0)
    if "N" in meta and meta["N"] != samples.size:
        raise SignalParseError(f"metadata declares N={meta['N']} but file holds {samples.size} rows")
    if not duration > 0:
        raise SignalParseError(f"duration must be positive, got {duration}")
    return Signal(samples, duration)


def read_signal_json(path) -> Signal:
    try:
        obj = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise SignalParseError(exc.msg, exc.lineno) from None
    if not isinstance(obj, dict):
        raise SignalParseError("top-level JSON value must be an object", 1)
    T = obj.get("T")
    if "samples" in obj:
        seq = obj["samples"]
        if not isinstance(seq, list) or not seq:
            raise SignalParseError("'samples' must be a non-empty list", 1)

        def one(i, e):
            if isinstance(e, (int, float)) and not isinstance(e, bool):
                return complex(e, 0.0)
            if isinstance(e, list) and len(e) == 2 and all(isinstance(v, (int, float)) for v in e):
                return complex(e[0], e[1])
            raise SignalParseError(f"sample {i} must be a number or [re, im] pair", 1)

        return Signal(np.array([one(i, e) for i, e in enumerate(seq)]), 1.0 if T is None else T)
    if "time" in obj and "value" in obj:
        t, v = obj["time"], obj["value"]
        if not isinstance(t, list) or not isinstance(v, list) or len(t) != len(v) or not t:
            raise SignalParseError("'time' and 'value' must be equal-length non-empty lists", 1)
        derived = _uniform_duration(t, 1)
        if T is None:
            T = derived if derived is not None else 1.0
        return Signal(np.asarray(v, dtype=float), T)
    raise SignalParseError("JSON object needs either 'samples' or 'time'+'value'", 1)


def read_signal(path) -> Signal:
    return read_signal_json(path) if Path(path).suffix.lower() == ".json" else read_signal_csv(path)


def write_signal_csv(signal: Signal, path) -> None:
    out = [f"# T={fmt17(signal.duration)}", f"# N={len(signal)}", "index,re,im"]
    out += [f"{i},{fmt17(z.real)},{fmt17(z.imag)}" for i, z in enumerate(signal.samples)]
    Path(path).write_text("\n".join(out) + "\n")


def write_spectrum(spectrum: Spectrum, path, method: str) -> None:
    out = [f"# N={spectrum.origin_n}", f"# alpha={spectrum.alpha.p}/{spectrum.alpha.q}",
           f"# T={fmt17(spectrum.duration)}", f"# method={method}", "m,freq,re,im,magnitude"]
    for m, z in enumerate(spectrum.bins):
        out.append(f"{m},{fmt17(bin_frequency(m, spectrum.alpha, spectrum.duration))},{fmt17(z.real)},"
                   f"{fmt17(z.imag)},{fmt17(abs(z))}")
    Path(path).write_text("\n".join(out) + "\n")


def read_spectrum(path) -> tuple:
    meta, rows = _csv_rows(path)
    if not rows:
        raise SignalParseError("no spectrum rows found")
    (hline, header), body = rows[0], rows[1:]
    if [c.lower() for c in header] != ["m", "freq", "re", "im", "magnitude"]:
        raise SignalParseError(f"expected header 'm,freq,re,im,magnitude', got {','.join(header)!r}", hline)
    bins = []
    for line_no, cells in body:
        if len(cells) != 5:
            raise SignalParseError(f"expected 5 columns, got {len(cells)}", line_no)
        try:
            m = int(cells[0])
        except ValueError:
            raise SignalParseError(f"expected an integer bin index, got {cells[0]!r}", line_no) from None
        if m != len(bins):
            raise SignalParseError(f"bin index {m} out of order (expected {len(bins)})", line_no)
        bins.append(complex(_num(cells[2], line_no), _num(cells[3], line_no)))
    for key in ("N", "alpha", "T"):
        if key not in meta:
            raise SignalParseError(f"missing '# {key}=' metadata")
    if not bins:
        raise SignalParseError("no spectrum rows found")
    n, alpha = meta["N"], meta["alpha"]
    full = n * alpha.p % alpha.q == 0 and len(bins) == n * alpha.p // alpha.q
    spec = Spectrum(np.asarray(bins), n, alpha, meta["T"], m_bins=None if full else len(bins))
    return spec, meta.get("method", "unknown")
