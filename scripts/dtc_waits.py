#!/usr/bin/env python
"""Wait accounting of k_direct_tc's roles (variant build -DASX_DTC_WAITS via
ASX_LIB_PATH): cycles CTA 0's role threads spend in each mbarrier wait."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate_device

w = WORKLOADS["3"]
batch = w.batch
x = generate_device(w, 0, batch, device="cuda")
p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method="auto")
big = torch.zeros((batch + 1, w.m), dtype=getattr(torch, w.dtype), device="cuda")
for _ in range(3):
    p.execute(x, out=big[:batch])
torch.cuda.synchronize()
d = big[batch].view(torch.int64).cpu().numpy()
print("converter (warp 0): wait sc_full %d, a_empty %d, acc_full %d, epilogue (incl. acc_full) %d, total %d, tiles %d" % tuple(d[[0, 1, 2, 3, 4, 5]]))
print("CTA 0 wall %d ns -> SM clock %.0f MHz" % (d[6], d[4] / max(d[6], 1) * 1e3))
print("epilogue: tcgen05.ld + wait %d cycles" % d[7])
print("MMA issuer: wait acc_empty %d, a_full %d, b_full %d, total %d, tiles %d" % tuple(d[[8, 9, 10, 12, 13]]))
print("scale warp 10: wait sc_empty %d, total %d, tiles %d" % tuple(d[[16, 20, 21]]))
print("W loader: wait b_empty %d, total %d, parts %d" % tuple(d[[24, 28, 29]]))
