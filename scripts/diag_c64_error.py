"""Find config-4 signals where the two GPU methods disagree most; compare each with the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate_device
from oracle import alpha_oracle as orc

w = WORKLOADS["4"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = generate_device(w, 0, B, device="cuda")
res = {}
for meth in ("chirp", "fft"):
    p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=meth)
    res[meth] = p.execute(x)
d = ((res["chirp"] - res["fft"]).abs().amax(dim=1) / res["fft"].abs().amax(dim=1))
top = torch.topk(d, 4).indices.cpu().numpy()
print("max chirp-vs-fft", d.max().item(), "median", d.median().item(), "top", top)
xs = x[torch.from_numpy(top).cuda()].cpu().numpy()
want = orc.alpha_fft(xs.astype(np.complex128), 1, 8, w.m)
for meth in ("chirp", "fft"):
    got = res[meth][torch.from_numpy(top).cuda()].cpu().numpy().astype(np.complex128)
    for i in range(len(top)):
        err = np.abs(got[i] - want[i])
        j = int(np.argmax(err))
        print(meth, "sig", top[i], "rel", err.max() / np.abs(want[i]).max(), "argmax bin", j,
              "|X| there", abs(want[i][j]), "max|X|", np.abs(want[i]).max(), "rms err", np.sqrt(np.mean(err**2)))
