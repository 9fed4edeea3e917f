"""PCIe ceiling on the GPU box: pinned H2D / D2H alone and concurrent (python tools/probe/pcie_probe.py)."""
import time

import torch

n = 4_697_948_160 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
m = 1_879_179_264 // 8
ho = torch.empty(m, dtype=torch.float64, pin_memory=True)
do = torch.empty(m, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: ho.copy_(do, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    nb = (h if name == "h2d" else ho).numel() * 8
    print(f"{name} {nb / 1e9:.2f} GB {dt * 1e3:.1f} ms {nb / dt / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"concurrent h2d 4.70 GB + d2h 1.88 GB: {dt * 1e3:.1f} ms")
