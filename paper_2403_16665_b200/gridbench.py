"""The reference's operation-count / wall-time grid and its scaling claims,
on GPU plans (ref/bench.py:1-422).

Same record, verdict and report schema as the reference, so a consumer of
``alpha-spectra bench`` JSON / CSV reads ours unchanged:

* ``BenchRecord.to_row`` -> ``N, alpha_p, alpha_q, method, mults, adds,
  wall_ns, reps`` (ref/bench.py:63-73, CSV columns :126-134);
* ``ScalingReport.to_dict`` -> ``{"records", "verdicts", "skipped"}`` with
  verdicts ``{"claim", "pass", "record_ids", "details", "warnings"}``
  (ref/bench.py:85-93, :103-116);
* claims ``alpha_gt1_savings``, ``alpha_lt1_savings`` and
  ``complexity_fit_alpha_<p>_<q>`` (ref/bench.py:279-422).

What differs is where the time comes from: each cell is one transform of one
signal on the B200 -- the α-FFT plan (method ``fft``), the α = 1 FFT of the
zero-padded signal (padding done on the device inside the timed region, as
the reference pads inside its timed closure, ref/bench.py:184-193), or the
direct form -- timed with CUDA events on the launch stream, minimum over
``reps`` (the reference's min-of-reps convention, ref/bench.py:159-167), plan
construction untimed.  Counts are the exact closed forms the reference's
instrumented runs produce (ref/fastpath.py:113-127, ref/bench.py:195-199);
they do not depend on the data, so the claims are integer identities.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field

import numpy as np

from .core import DenseFactor, IncompatibleAlphaError, is_power_of_two, validate_pair

METHODS = ("alpha_fft", "zeropad_fft", "naive")
ROW_FIELDS = ("N", "alpha_p", "alpha_q", "method", "mults", "adds", "wall_ns", "reps")


class IncompleteGridError(ValueError):
    """A claim needs grid points the record set does not contain."""


@dataclass(frozen=True)
class BenchRecord:
    """One (N, alpha, method) cell: exact counts and the best device time (s)."""

    n: int
    alpha: DenseFactor
    method: str
    complex_mults: int
    complex_adds: int
    wall_time: float
    repetitions: int

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if min(self.complex_mults, self.complex_adds) < 0:
            raise ValueError("operation counts cannot be negative")
        if not (self.wall_time > 0 and self.repetitions >= 1):
            raise ValueError("wall_time must be positive and repetitions >= 1")

    def to_row(self) -> dict:
        vals = (self.n, self.alpha.p, self.alpha.q, self.method, self.complex_mults, self.complex_adds,
                int(round(self.wall_time * 1e9)), self.repetitions)
        return dict(zip(ROW_FIELDS, vals))


@dataclass
class ClaimVerdict:
    claim: str
    passed: bool
    record_ids: list = field(default_factory=list)
    details: list = field(default_factory=list)
    warnings: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {"claim": self.claim, "pass": self.passed, "record_ids": self.record_ids,
                "details": self.details, "warnings": self.warnings}


@dataclass
class FitResult:
    c: float
    max_rel_residual: float
    passed: bool
    n_points: int
    record_ids: list = field(default_factory=list)


def write_records_csv(records, path) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.DictWriter(fh, fieldnames=list(ROW_FIELDS))
        out.writeheader()
        out.writerows(r.to_row() for r in records)


@dataclass
class ScalingReport:
    records: list
    verdicts: list
    skipped: list = field(default_factory=list)

    @property
    def all_passed(self) -> bool:
        return all(v.passed for v in self.verdicts)

    def to_dict(self) -> dict:
        return {"records": [r.to_row() for r in self.records], "verdicts": [v.to_dict() for v in self.verdicts],
                "skipped": list(self.skipped)}

    def write_json(self, path) -> None:
        with open(path, "w") as fh:
            fh.write(json.dumps(self.to_dict(), indent=2) + "\n")

    def write_csv(self, path) -> None:
        write_records_csv(self.records, path)


def _lg(v: int) -> int:
    return v.bit_length() - 1


def cell_validity(n: int, alpha: DenseFactor, method: str) -> tuple[bool, str]:
    """(runnable, reason) of a grid cell under the reference's rules (ref/bench.py:141-156)."""
    if method not in METHODS:
        return False, f"unknown method {method!r}"
    try:
        m = validate_pair(n, alpha).m
    except IncompatibleAlphaError:
        return False, f"alpha*N = {alpha.p * n}/{alpha.q} is not an integer"
    if method == "alpha_fft" and not (is_power_of_two(n) and is_power_of_two(m)):
        return False, f"N={n}, alpha*N={m} not both powers of two"
    if method == "zeropad_fft" and alpha.p < alpha.q:
        return False, "zero-padding needs alpha >= 1"
    if method == "zeropad_fft" and not is_power_of_two(m):
        return False, f"padded length {m} not a power of two"
    return True, ""


def cell_counts(n: int, alpha: DenseFactor, method: str) -> tuple[int, int]:
    """Exact complex (mults, adds) of one transform, as the reference's counter tallies them."""
    m = validate_pair(n, alpha).m
    if method == "naive":  # the matrix product: N M multiplies, (N-1) M adds
        return n * m, (n - 1) * m
    if method == "zeropad_fft":  # the alpha = 1 recursion over the padded length m
        return (m // 2) * _lg(m), m * _lg(m)
    depth = _lg(min(n, m))
    return (m // 2) * depth, m * depth + max(n - m, 0)


def _unit_disk_signals(ns, seed):
    """One complex unit-disk signal per distinct N, drawn in sorted-N order from one seed."""
    rng = np.random.default_rng(seed)
    out = {}
    for n in sorted(set(ns)):
        r = np.sqrt(rng.uniform(0.0, 1.0, n))
        out[n] = r * np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, n))
    return out


def _device_timer(n, alpha, method, x):
    """Untimed plan + upload; returns run() -> device seconds of one transform."""
    import torch

    from .transforms import plan

    m = validate_pair(n, alpha).m
    dev = torch.cuda.current_device()
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{dev}")
    if method == "alpha_fft":
        p = plan(n, alpha, method="fft")

        def body():
            p.execute(xd)
    elif method == "zeropad_fft":
        p = plan(m, DenseFactor(1), method="fft")

        def body():
            buf = torch.zeros(m, dtype=torch.complex128, device=xd.device)
            buf[:n] = xd
            p.execute(buf)
    else:
        p = plan(n, alpha, method="direct")

        def body():
            p.execute(xd)

    stream = torch.cuda.current_stream(xd.device)
    body()  # warm-up (lazy module loads, workspace)
    torch.cuda.synchronize()

    def run() -> float:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        body()
        e.record(stream)
        e.synchronize()
        return max(s.elapsed_time(e) * 1e-3, 1e-9)

    return run


def grid_cells(ns, alphas, methods, skipped: list | None = None) -> list:
    """Runnable (N, alpha, method) cells in grid order; the others go to ``skipped``
    as dicts with N, alpha_p, alpha_q, method, reason."""
    cells = []
    for n in ns:
        for alpha in alphas:
            for method in methods:
                ok, why = cell_validity(n, alpha, method)
                if ok:
                    cells.append((n, alpha, method))
                elif skipped is not None:
                    skipped.append({"N": n, "alpha_p": alpha.p, "alpha_q": alpha.q, "method": method, "reason": why})
    return cells


def run_grid(ns, alphas, methods=("alpha_fft", "zeropad_fft"), reps: int = 20, naive_reps: int = 3, seed: int = 0,
             skipped: list | None = None) -> list:
    """One BenchRecord per runnable (N, alpha, method) cell, in grid order (ref/bench.py:210-265).

    Invalid cells are collected in ``skipped`` instead of failing the grid.
    """
    signals = _unit_disk_signals(ns, seed)
    records = []
    for n, alpha, method in grid_cells(ns, alphas, methods, skipped):
        mults, adds = cell_counts(n, alpha, method)
        k = min(reps, naive_reps) if method == "naive" else reps
        run = _device_timer(n, alpha, method, signals[n])
        best = min(run() for _ in range(k))
        records.append(BenchRecord(n, alpha, method, mults, adds, best, k))
    return records


def _cells(records):
    return {(r.n, r.alpha, r.method): (i, r) for i, r in enumerate(records)}


def check_alpha_gt1_savings(records) -> ClaimVerdict:
    """alpha > 1: zeropad_mults - alpha_mults == (alpha N / 2) log2(alpha), exactly (ref/bench.py:279-311)."""
    cells = _cells(records)
    v = ClaimVerdict("alpha_gt1_savings", True)
    pairs = sorted(((i, r, cells.get((r.n, r.alpha, "zeropad_fft"))) for (_, _, meth), (i, r) in cells.items()
                    if meth == "alpha_fft" and r.alpha.p > r.alpha.q), key=lambda t: t[0])
    for i, fast, pad in pairs:
        if pad is None:
            continue
        j, padded = pad
        m = validate_pair(fast.n, fast.alpha).m
        want = (m // 2) * _lg(fast.alpha.p // fast.alpha.q)
        gap = padded.complex_mults - fast.complex_mults
        ok = gap > 0 and gap == want
        v.passed = v.passed and ok
        v.record_ids.extend([i, j])
        v.details.append({"N": fast.n, "alpha": str(fast.alpha), "zeropad_mults": padded.complex_mults,
                          "alpha_mults": fast.complex_mults, "gap": gap, "expected_gap": want, "ok": ok})
    if not v.details:
        raise IncompleteGridError("no (alpha_fft, zeropad_fft) record pairs with alpha > 1 in the grid")
    return v


def check_alpha_lt1_savings(records, min_m: int = 16) -> ClaimVerdict:
    """alpha < 1 vs alpha = 1 at the same N: gap == (N/2)log2 N - (M/2)log2 M, >= (N/2)log2(1/alpha)
    (ref/bench.py:314-353); cells with M < min_m are warnings, not judged."""
    cells = _cells(records)
    v = ClaimVerdict("alpha_lt1_savings", True)
    unit = DenseFactor(1)
    for (_, _, meth), (i, fast) in sorted(cells.items(), key=lambda kv: kv[1][0]):
        if meth != "alpha_fft" or fast.alpha.p >= fast.alpha.q:
            continue
        full = cells.get((fast.n, unit, "alpha_fft"))
        if full is None:
            continue
        n, m = fast.n, validate_pair(fast.n, fast.alpha).m
        if m < min_m:
            v.warnings.append(f"N={n}, alpha={fast.alpha}: alpha*N={m} < {min_m}, excluded from the claim")
            continue
        j, whole = full
        want = (n // 2) * _lg(n) - (m // 2) * _lg(m)
        floor = (n // 2) * _lg(fast.alpha.q // fast.alpha.p)
        gap = whole.complex_mults - fast.complex_mults
        ok = gap == want and gap >= floor
        v.passed = v.passed and ok
        v.record_ids.extend([i, j])
        v.details.append({"N": n, "alpha": str(fast.alpha), "fft_mults": whole.complex_mults,
                          "alpha_mults": fast.complex_mults, "gap": gap, "expected_gap": want, "floor": floor,
                          "ok": ok})
    if not (v.details or v.warnings):
        raise IncompleteGridError("need alpha < 1 alpha_fft records plus the alpha = 1 record at the same N")
    return v


def fit_complexity(records, residual_limit: float = 0.01) -> FitResult:
    """Least squares of mults against max(N, M) log2 min(N, M) through the origin (ref/bench.py:356-381)."""
    rows = []
    for i, r in enumerate(records):
        m = validate_pair(r.n, r.alpha).m
        lo = min(r.n, m)
        if lo > 1:
            rows.append((i, r.n, max(r.n, m) * _lg(lo), r.complex_mults))
    if len({n for _, n, _, _ in rows}) < 4:
        raise IncompleteGridError("complexity fit needs at least 4 distinct N values")
    f = np.array([row[2] for row in rows], dtype=float)
    y = np.array([row[3] for row in rows], dtype=float)
    c = float(np.dot(f, y) / np.dot(f, f))
    resid = float(np.max(np.abs(y - c * f) / y))
    return FitResult(c, resid, resid <= residual_limit, len(rows), [row[0] for row in rows])


def make_report(records, skipped: list | None = None) -> ScalingReport:
    """Every evaluable claim on a record set; claims without their grid points are left out (ref/bench.py:384-422)."""
    verdicts = []
    for check in (check_alpha_gt1_savings, check_alpha_lt1_savings):
        try:
            verdicts.append(check(records))
        except IncompleteGridError:
            pass
    groups: dict = {}
    for r in records:
        if r.method == "alpha_fft":
            groups.setdefault(r.alpha, []).append(r)
    for alpha in sorted(groups, key=lambda a: (a.p / a.q, a.p)):
        try:
            fit = fit_complexity(groups[alpha])
        except IncompleteGridError:
            continue
        expected = 0.5 * (alpha.p / alpha.q) if alpha.p < alpha.q else 0.5
        verdicts.append(ClaimVerdict(f"complexity_fit_alpha_{alpha.p}_{alpha.q}", fit.passed,
                                     [records.index(r) for r in groups[alpha]],
                                     [{"c": fit.c, "expected_c": expected, "max_rel_residual": fit.max_rel_residual,
                                       "n_points": fit.n_points}]))
    return ScalingReport(list(records), verdicts, list(skipped or []))
