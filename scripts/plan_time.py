import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_16665_b200 as asx
torch.cuda.init(); asx.plan(64, asx.DenseFactor(2))
for (n, d, dt) in [(8192, 8, "complex64"), (4096, 10, "complex128"), (256, 1, "complex64"), (1 << 22, 16, "complex128")]:
    t0 = time.perf_counter(); p = asx.plan(n, asx.DenseFactor(d), m=n, dtype=dt, method="chirp"); dtm = time.perf_counter() - t0
    print(f"plan N={n} d={d} {dt}: {dtm*1e3:.1f} ms (P={p.fft_size})")
