"""Per-signal complex64 error of config-4 signals (GPU inputs saved for CPU
emulation): python scripts/diag_c64_signals.py idx [idx ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate_device

w = WORKLOADS["4"]
idx = [int(a) for a in sys.argv[1:]]
xs = torch.cat([generate_device(w, i, 1, device="cuda") for i in idx])
ref = asx.plan(w.n, w.density, m=w.m, dtype="complex128", method="chirp").execute(xs.to(torch.complex128))
got = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method="chirp").execute(xs).to(torch.complex128)
err = ((got - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)).cpu().numpy()
for i, e in zip(idx, err):
    print(i, f"{e:.3e}")
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/diag_signals.npz", idx=np.array(idx), x=xs.cpu().numpy(), got=got.cpu().numpy(),
         ref=ref.cpu().numpy())
