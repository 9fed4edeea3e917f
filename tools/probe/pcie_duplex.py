"""PCIe full-duplex ceiling on the GPU box: equal page-locked H2D and D2H streams alone and
concurrently (python tools/probe/pcie_duplex.py) -- the floor of the config 5 e2e leg, which
moves 33.4 GB up and 45.1 GB down per sweep."""
import time

import torch

n = (4 << 30) // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
ho = torch.empty(n, dtype=torch.float64, pin_memory=True)
do = torch.empty(n, dtype=torch.float64, device="cuda")
h.zero_(); ho.zero_()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = n * 8


def run(up, down, reps=4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if up:
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if down:
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for name, up, down in (("h2d alone", 1, 0), ("d2h alone", 0, 1), ("h2d + d2h concurrent", 1, 1)):
    run(up, down, 1)
    dt = run(up, down)
    tot = nb * (up + down)
    print(f"{name}: {tot / 1e9:.2f} GB in {dt * 1e3:.1f} ms = {tot / dt / 1e9:.1f} GB/s total"
          + (f" ({nb / dt / 1e9:.1f} GB/s per direction)" if up and down else ""))
