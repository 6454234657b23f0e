#!/usr/bin/env python
"""Device-time sweep over BASELINE configs x methods (CUDA events, after warm-up).

    python scripts/sweep.py [--configs 0,1a,1b,3,4] [--methods fft,chirp,direct] [--reps 10]

Prints one JSON object per (config, method) with ms, points/s, HBM fraction
of the algorithmic bytes and the reference closed-form FLOP rate.
"""

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1a,1b,3,4")
    ap.add_argument("--methods", default="fft,chirp,direct")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    import torch

    import paper_2403_16665_b200 as asx
    from paper_2403_16665_b200.signals import WORKLOADS, generate_device

    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    for key in args.configs.split(","):
        w = WORKLOADS[key]
        batch = args.batch or w.batch
        x = generate_device(w, 0, batch, device="cuda")
        for method in args.methods.split(","):
            try:
                p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=method, real_input=w.real)
            except Exception as exc:  # unsupported combination
                print(json.dumps({"config": key, "method": method, "skip": str(exc)[:120]}), flush=True)
                continue
            if method == "direct" and w.n * w.m * batch > 2e13:
                print(json.dumps({"config": key, "method": method, "skip": "too slow"}), flush=True)
                continue
            out = torch.empty((batch, w.m), dtype=getattr(torch, w.dtype), device="cuda")
            for _ in range(3):
                p.execute(x, out=out)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.reps):
                p.execute(x, out=out)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / args.reps
            import ctypes
            from paper_2403_16665_b200 import _lib
            sh = [ctypes.c_int() for _ in range(4)]
            _lib.lib().asx_last_launch(*[ctypes.byref(v) for v in sh])
            shape = dict(zip(("grid", "block", "smem", "staged"), (v.value for v in sh)))
            gbs = w.bytes_alg(batch) / (ms / 1e3) / 1e9
            print(json.dumps({"config": key, "method": method, "fft_size": p.fft_size, "batch": batch,
                              "ms": round(ms, 4), "points_per_s": batch * w.m / (ms / 1e3),
                              "hbm_frac": round(gbs / peak, 4), "gbs": round(gbs, 1),
                              "alg_tflops": round(w.flops_alg(batch) / (ms / 1e3) / 1e12, 2), **shape}), flush=True)
            del out
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
