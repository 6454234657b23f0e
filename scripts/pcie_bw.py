#!/usr/bin/env python
"""Host<->device copy bandwidth from pinned memory (the e2e roofline).

    python scripts/pcie_bw.py [--mib 1024] [--reps 5]

Prints JSON: H2D alone, D2H alone, and both directions at once on two streams
(what a pipelined host-buffer execute overlaps), in GB/s (1e9 B/s).
"""

import argparse
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    n = args.mib << 20
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    h_in.fill_(1)
    d_out.fill_(2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = 1e30
        for _ in range(args.reps + 1):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            # join both side streams into the timing stream
            cur = torch.cuda.current_stream()
            cur.wait_stream(s1)
            cur.wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return best

    def h2d():
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({
        "bytes": n, "h2d_gbs": n / t_h2d / 1e9, "d2h_gbs": n / t_d2h / 1e9,
        "duplex_total_gbs": 2 * n / t_both / 1e9, "duplex_per_direction_gbs": n / t_both / 1e9,
        "how": f"pinned {args.mib} MiB torch copies, best of {args.reps}, CUDA events",
    }))


if __name__ == "__main__":
    main()
