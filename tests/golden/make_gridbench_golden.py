"""Golden report of the REFERENCE's bench grid (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_gridbench_golden.py

Runs the reference's own run_grid + make_report (ref/bench.py:210-422),
imported read-only from /root/reference/pkg/src, on a grid that exercises
every claim and skip reason, and writes the report (records, verdicts,
skipped) and its CSV to tests/golden/gridbench_ref.{json,csv}.  Wall times
are data-independent of the checks; tests/test_gridbench.py compares our
counts, skips, verdicts and the exact JSON / CSV layout against these files.
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from alpha_spectra import DenseFactor  # noqa: E402  (the reference, read-only)
from alpha_spectra.bench import make_report, run_grid  # noqa: E402

NS = [6, 64, 128, 256, 512]
ALPHAS = [(1, 8), (1, 4), (1, 2), (1, 1), (3, 2), (2, 1), (4, 1), (8, 1)]
METHODS = ("alpha_fft", "zeropad_fft", "naive")


def main():
    skipped = []
    recs = run_grid(NS, [DenseFactor(p, q) for p, q in ALPHAS], METHODS, reps=1, naive_reps=1, seed=0,
                    skipped=skipped)
    rep = make_report(recs, skipped)
    with open(os.path.join(HERE, "gridbench_ref.json"), "w") as fh:
        json.dump({"grid": {"ns": NS, "alphas": ALPHAS, "methods": list(METHODS)}, "report": rep.to_dict()}, fh,
                  indent=1)
        fh.write("\n")
    rep.write_csv(os.path.join(HERE, "gridbench_ref.csv"))


if __name__ == "__main__":
    main()
