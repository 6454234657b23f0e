"""Host-buffer path (asx_execute_host) throughput vs chunk size, config 4."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_16665_b200 as asx
from paper_2403_16665_b200.signals import WORKLOADS, generate_device
w = WORKLOADS["4"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
x = generate_device(w, 0, B, device="cuda")
hx = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); hx.copy_(x)
hX = torch.empty((B, w.m), dtype=x.dtype, pin_memory=True)
p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype)
for rows in [int(r) for r in (sys.argv[2].split(",") if len(sys.argv) > 2 else (0, 128, 256, 512, 1024, 2048))]:
    p.execute_host(hx.numpy(), out=hX.numpy(), chunk=rows)
    t0 = time.perf_counter()
    for _ in range(3):
        p.execute_host(hx.numpy(), out=hX.numpy(), chunk=rows)
    el = (time.perf_counter() - t0) / 3
    gb = B * w.n * 8 * 2 / 1e9
    print(f"chunk {rows:5d} rows: {el*1e3:8.2f} ms  {gb/el:6.1f} GB/s (H2D+D2H)  -> full batch ~{el*w.batch/B*1e3:.1f} ms", flush=True)
