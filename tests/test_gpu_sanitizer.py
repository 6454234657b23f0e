"""compute-sanitizer over the hot kernels (race detection).

The kernels rely on split-phase mbarriers (write-after-read protection of
exchange buffers), "each thread rewrites exactly the slots it read" local
exchanges, TMA bulk copies into shared memory (async proxy) and tensor
memory; racecheck and synccheck check the shared-memory hazards and barrier
use on small batches of each (tests/sanitize_driver.py), memcheck the
bounds on ragged sizes, odd batches and strided rows.  Pass = the tool's
ERROR SUMMARY reports 0 errors and the driver exits 0."""

import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool, mode", [("racecheck", "all"), ("synccheck", "all"), ("memcheck", "ragged"),
                                        ("memcheck", "all")])
def test_sanitizer_clean(tool, mode):
    assert os.path.exists(SAN), "compute-sanitizer not found"
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=99", "--print-limit=20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report=all"]
    r = subprocess.run(cmd + [sys.executable, os.path.join(HERE, "sanitize_driver.py"), mode], capture_output=True,
                       text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", r.stdout + r.stderr)
    assert m is not None, tail
    assert int(m.group(1)) == 0 and r.returncode == 0, tail
    assert r.stdout.count("ok ") >= 5, tail
