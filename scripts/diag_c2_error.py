import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate
from oracle import alpha_oracle as orc
w = WORKLOADS["2"]
x = generate(w, 0, 1)[0]
want = np.fft.fft(x, 16 * w.n)[: w.m]
for method in ("chirp", "fft"):
    p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=method, real_input=True)
    got = p.execute(torch.from_numpy(x[None]).cuda()).cpu().numpy()
    print(method, "rel_err", orc.rel_err(got, want[None]))
