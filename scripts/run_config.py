#!/usr/bin/env python
"""Run one BASELINE config's transform a few times (the short command to put
under ncu): python scripts/run_config.py --config 3 [--method auto] [--reps 3]"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3")
    ap.add_argument("--method", default="auto")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    import torch

    import paper_2403_16665_b200 as asx
    from paper_2403_16665_b200.signals import WORKLOADS, generate_device

    w = WORKLOADS[args.config]
    batch = args.batch or w.batch
    x = generate_device(w, 0, batch, device="cuda")
    p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=args.method, real_input=w.real)
    out = torch.empty((batch, w.m), dtype=getattr(torch, w.dtype), device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(args.reps):
        s.record()
        p.execute(x, out=out)
        e.record()
        torch.cuda.synchronize()
        print(f"config {args.config} {p.method}: {s.elapsed_time(e):.4f} ms", flush=True)


if __name__ == "__main__":
    main()
