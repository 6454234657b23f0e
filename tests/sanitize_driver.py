"""Small launches of every hot kernel, run under compute-sanitizer by
tests/test_gpu_sanitizer.py (not collected by pytest: no test_ prefix).

    python tests/sanitize_driver.py [all|ragged]

`all` runs each production kernel once on a small batch (a few signals, so
racecheck / synccheck finish in seconds); `ragged` runs them on odd batch
sizes, ragged N / M and strided rows, for memcheck's bounds checks.
"""

import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2403_16665_b200 as asx  # noqa: E402

# (label, n, alpha_b = a/d, m, dtype, method, batch): the kernel each one launches
CASES = [
    ("k_chirp_local", 8192, 1, 8, 8192, "complex64", "chirp", 3),
    ("k_afft_local", 4096, 1, 2, 4096, "complex128", "fft", 3),
    ("k_chirp_local128", 4096, 1, 10, 4096, "complex128", "chirp", 3),
    ("k_direct_tc", 256, 37, 100, 256, "complex64", "direct", 130),
    ("k_fft_persist alpha-FFT (FP64 recursion, complex64 I/O)", 1024, 1, 4, 1024, "complex64", "fft", 5),
    ("k_fft_persist chirp", 256, 37, 100, 256, "complex64", "chirp", 5),
    ("four-step chirp", 8192, 1, 8, 8192, "complex128", "chirp", 1),
]
RAGGED = [
    ("k_chirp_local ragged", 6000, 1, 8, 7001, "complex64", "chirp", 5),
    ("k_afft_local M < N", 4096, 1, 2, 3001, "complex128", "fft", 5),
    ("k_chirp_local128 ragged", 3001, 1, 10, 4000, "complex128", "chirp", 5),
    ("k_direct_tc ragged tile", 96, 2, 3, 256, "complex64", "direct", 131),
    ("alpha-FFT block-sum leaf", 1024, 4, 1, 256, "complex128", "fft", 7),
]


def run(cases, strided):
    rng = np.random.default_rng(0)
    for label, n, a, d, m, dtype, method, batch in cases:
        p = asx.plan(n, asx.DenseFactor(d, a), m=m, dtype=dtype, method=method)
        cdt = getattr(torch, dtype)
        pad = 3 if strided else 0  # rows inside a wider buffer (odd stride: unaligned rows)
        buf = torch.from_numpy((rng.standard_normal((batch, n + pad)) + 1j * rng.standard_normal((batch, n + pad)))
                               .astype(np.complex64 if dtype == "complex64" else np.complex128)).cuda()
        x = buf[:, :n]
        out = torch.empty((batch, m + pad), dtype=cdt, device="cuda")[:, :m]  # strided output rows too
        y = p.execute(x, out=out)
        torch.cuda.synchronize()
        assert bool(torch.isfinite(torch.view_as_real(y)).all()), label
        print(f"ok {label}", flush=True)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    if mode == "all":
        run(CASES, strided=False)
    else:
        run(RAGGED, strided=False)
        run(RAGGED, strided=True)
