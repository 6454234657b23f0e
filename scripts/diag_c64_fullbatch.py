"""Per-signal error of the complex64 methods over the full config-4 batch, against the
complex128 GPU path (itself parity-tested to 1e-10) on the same inputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate_device

w = WORKLOADS["4"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else w.batch
x = generate_device(w, 0, B, device="cuda")
ref = asx.plan(w.n, w.density, m=w.m, dtype="complex128", method="chirp")
res = {m: asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=m) for m in ("chirp", "fft")}
errs = {m: [] for m in res}
for b0 in range(0, B, 4096):
    xb = x[b0:b0 + 4096]
    want = ref.execute(xb.to(torch.complex128))
    scale = want.abs().amax(dim=1)
    for m, p in res.items():
        got = p.execute(xb).to(torch.complex128)
        errs[m].append(((got - want).abs().amax(dim=1) / scale).cpu())
for m in errs:
    e = torch.cat(errs[m]).numpy()
    print(m, "max", e.max(), "p99.9", np.quantile(e, 0.999), "median", np.median(e), "worst idx", int(e.argmax()), flush=True)
