#!/usr/bin/env python
"""Phase timeline of one CTA of a hot kernel (variant builds with
-DASX_AFL_TIMELINE=<it> / -DASX_CL_TIMELINE=<it>; ASX_LIB_PATH selects the
library): prints, per warp, the clock64() deltas between phase stamps of two
consecutive signals.  python scripts/timeline.py --config 1a|4 [--batch B]"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1a")
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2403_16665_b200 as asx
    from paper_2403_16665_b200.signals import WORKLOADS, generate_device

    w = WORKLOADS[args.config]
    batch = args.batch or min(w.batch, 8192)
    x = generate_device(w, 0, batch, device="cuda")
    p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method="auto", real_input=w.real)
    big = torch.zeros((batch + 1, w.m), dtype=getattr(torch, w.dtype), device="cuda")
    for _ in range(3):
        p.execute(x, out=big[:batch])
    torch.cuda.synchronize()
    nw, ns = (16, 16) if args.config.startswith("1") else (32, 32)
    raw = big[batch].view(torch.int64).cpu().numpy()[: 2 * nw * ns].reshape(2, nw, ns)
    t0 = raw[0][raw[0] > 0].min()
    np.set_printoptions(linewidth=250)
    for it in range(2):
        print(f"iteration {it}: stamps relative to the CTA's first stamp (cycles), rows = warps")
        for wi in range(nw):
            row = raw[it, wi]
            n = int((row > 0).sum())
            print(f"w{wi:02d} " + " ".join(f"{int(v - t0):6d}" for v in row[:n]))
    print("period (warp 0, stamp 0):", int(raw[1, 0, 0] - raw[0, 0, 0]))
    d = np.diff(raw[0].astype(np.int64), axis=1)
    n = int((raw[0, 0] > 0).sum())
    print("mean phase length over warps (stamp i -> i+1):")
    print(" ".join(f"{int(v):6d}" for v in d[:, : n - 1].mean(axis=0)))


if __name__ == "__main__":
    main()
