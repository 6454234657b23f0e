"""Accuracy of the config-4 methods on known worst-case signals + batch max over chirp-vs-fft."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate_device
from oracle import alpha_oracle as orc

w = WORKLOADS["4"]
idx = [15760, 18939, 47679, 44147, 48066, 5287, 5346]
x = torch.cat([generate_device(w, i, 1, device="cuda") for i in idx])
want = orc.alpha_fft(x.cpu().numpy().astype(np.complex128), 1, 8, w.m)
out = {"lib": os.path.basename(os.environ.get("ASX_LIB_PATH", "libasx.so"))}
for meth in ("chirp", "fft"):
    p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=meth)
    got = p.execute(x).cpu().numpy().astype(np.complex128)
    out[meth] = float(orc.rel_err(got, want))
print(out, flush=True)
