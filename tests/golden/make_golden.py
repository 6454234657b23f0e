"""Generate golden vectors from the REFERENCE implementation (run in the build container).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports the reference package ``alpha_spectra`` read-only from
/root/reference/pkg/src and records its outputs on seeded inputs into
tests/golden/*.npz / *.json.  The GPU box has no /root/reference, so these
committed fixtures are how the oracle (oracle/alpha_oracle.py) and the CUDA
path are pinned to the reference there.  Re-running must reproduce the files
bit for bit (numpy 2.3.5 / OpenBLAS 0.3.30 in this image).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import alpha_spectra as ref  # noqa: E402  (the reference, read-only)
from alpha_spectra.verify import random_unit_disk  # noqa: E402

from paper_2403_16665_b200 import signals  # noqa: E402  (pure-numpy generator only)

POWER_ALPHAS = [(1, 8), (1, 4), (1, 2), (1, 1), (2, 1), (4, 1), (8, 1)]
FFT_SIZES = [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024]
NAIVE_GRID_N = [1, 2, 3, 4, 6, 8, 12, 16]
NAIVE_GRID_PQ = [(1, 4), (1, 2), (2, 3), (1, 1), (3, 2), (2, 1), (3, 1), (4, 1)]


def kat() -> dict:
    out = {}
    out["two_sample_x"] = np.array([0.0, 1.0], dtype=np.complex128)
    out["two_sample_X"] = ref.naive_forward(ref.Signal([0.0, 1.0]), ref.DenseFactor(2)).bins
    rng = np.random.default_rng(3)
    x = random_unit_disk(rng, 4)
    out["halving_x"] = x
    out["halving_X"] = ref.naive_forward(ref.Signal(x), ref.DenseFactor(1, 2)).bins
    out["impulse_X"] = ref.alpha_fft(ref.Signal([1.0, 0.0, 0.0, 0.0]), ref.plan(4, ref.DenseFactor(2))).bins
    out["combine_id"] = ref.combine(np.array([1.0 + 0j]), np.array([1.0 + 0j]), np.array([1.0 + 0j]))
    out["combine_quarter"] = ref.combine(np.array([0j]), np.array([1.0 + 0j]), np.array([-1j]))
    rng = np.random.default_rng(11)
    y = random_unit_disk(rng, 24).reshape(3, 8)
    z = random_unit_disk(rng, 24).reshape(3, 8)
    tw = np.exp(-2j * np.pi * np.arange(8) / 16)
    out["combine_rows_y"], out["combine_rows_z"], out["combine_rows_tw"] = y, z, tw
    out["combine_rows_out"] = ref.combine(y, z, tw)
    rng = np.random.default_rng(2)
    block = random_unit_disk(rng, 8)
    out["block_x"] = block
    out["block_sum"] = np.array([ref.leaf_block_sum(block)])
    p = ref.plan(16, ref.DenseFactor(4))
    for k, t in enumerate(p.twiddles):
        out[f"twiddle_16_4_{k}"] = np.array(t)
    out["dft_matrix_12_2_3"] = ref.dft_matrix(12, ref.DenseFactor(2, 3))
    # inverse transform and comparators
    for (n, p, q) in [(8, 1, 1), (8, 2, 1), (16, 4, 1), (12, 3, 2), (16, 1, 4), (12, 1, 3), (64, 1, 1)]:
        rng = np.random.default_rng(1000 + n + 10 * p + q)
        x = random_unit_disk(rng, n)
        spec = ref.naive_forward(ref.Signal(x, duration=2.0), ref.DenseFactor(p, q))
        out[f"inv_n{n}_p{p}_q{q}_X"] = spec.bins
        out[f"inv_n{n}_p{p}_q{q}_x"] = ref.naive_inverse(spec).samples
        if p < q:
            out[f"alias_n{n}_p{p}_q{q}"] = ref.aliased_reconstruct(ref.Signal(x), ref.DenseFactor(p, q))
            out[f"alias_n{n}_p{p}_q{q}_in"] = x
    rng = np.random.default_rng(21)
    x = random_unit_disk(rng, 32)
    out["zeropad_x"] = x
    out["zeropad_X"] = ref.standard_fft(ref.zero_pad(ref.Signal(x), ref.DenseFactor(4))).bins
    out["orth_12_3_2"] = np.array([ref.orthogonality_kernel(d, 0, 12, ref.DenseFactor(3, 2)) for d in range(-11, 12)])
    return out


def grid_fft() -> dict:
    out = {}
    for n in FFT_SIZES:
        for (p, q) in POWER_ALPHAS:
            if (n * p) % q or n * p < q:
                continue
            alpha = ref.DenseFactor(p, q)
            pl = ref.plan(n, alpha)
            for s in range(2):
                x = random_unit_disk(np.random.default_rng(1000 * s + n), n)
                key = f"n{n}_p{p}_q{q}_s{s}"
                out[key + "_x"] = x
                out[key + "_fft"] = ref.transform_samples(x, pl)
                if n <= 256:
                    out[key + "_naive"] = ref.naive_forward(ref.Signal(x), alpha).bins
    return out


def grid_naive() -> dict:
    out = {}
    for n in NAIVE_GRID_N:
        for (p, q) in NAIVE_GRID_PQ:
            if (n * p) % q:
                continue
            rng = np.random.default_rng(100 * n + 10 * p + q)
            x = random_unit_disk(rng, n)
            key = f"n{n}_p{p}_q{q}"
            out[key + "_x"] = x
            out[key + "_naive"] = ref.naive_forward(ref.Signal(x), ref.DenseFactor(p, q)).bins
    return out


def configs() -> dict:
    out = {}
    w0 = signals.WORKLOADS["0"]
    x0 = signals.generate(w0, 0, 1)[0]
    out["c0_x"] = x0
    out["c0_naive"] = ref.naive_forward(ref.Signal(x0), ref.DenseFactor(4)).bins[:1024]
    out["c0_fft"] = ref.alpha_fft(ref.Signal(x0), ref.plan(1024, ref.DenseFactor(4))).bins[:1024]
    # config 1b in miniature: alpha_ref = 10 is rejected by the fast path, the
    # reference's own batched route is dft_matrix @ X (test_acceptance.py:64-67)
    rng = np.random.default_rng(7)
    X = np.column_stack([random_unit_disk(rng, 64) for _ in range(8)])
    out["c1b_mini_x"] = X.T.copy()
    out["c1b_mini_X"] = (ref.dft_matrix(64, ref.DenseFactor(10))[:64] @ X).T.copy()
    # config 4 in miniature: alpha_ref = 8, first N bins, signals upcast from c64
    rng = np.random.default_rng(8)
    x4 = np.stack([random_unit_disk(rng, 256) for _ in range(4)]).astype(np.complex64)
    pl = ref.plan(256, ref.DenseFactor(8))
    out["c4_mini_x"] = x4
    out["c4_mini_X"] = np.stack([ref.transform_samples(r.astype(np.complex128), pl)[:256] for r in x4])
    # config 1a in miniature
    rng = np.random.default_rng(9)
    x1 = np.stack([random_unit_disk(rng, 512) for _ in range(4)])
    pl = ref.plan(512, ref.DenseFactor(2))
    out["c1a_mini_x"] = x1
    out["c1a_mini_X"] = np.stack([ref.transform_samples(r, pl)[:512] for r in x1])
    return out


def counts() -> dict:
    rows = []
    for n in [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 4096, 8192]:
        for (p, q) in POWER_ALPHAS + [(16, 1)]:
            if (n * p) % q or n * p < q:
                continue
            pl = ref.plan(n, ref.DenseFactor(p, q))
            rows.append({"n": n, "p": p, "q": q, "m": pl.m, "depth": pl.depth, "leaf": pl.leaf.value,
                         "mults": ref.predicted_mults(pl), "adds": ref.predicted_adds(pl)})
    return {"rows": rows}


def main() -> None:
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kat())
    np.savez_compressed(os.path.join(HERE, "grid_fft.npz"), **grid_fft())
    np.savez_compressed(os.path.join(HERE, "grid_naive.npz"), **grid_naive())
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **configs())
    with open(os.path.join(HERE, "counts.json"), "w") as fh:
        json.dump(counts(), fh, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
