"""Host->device copy bandwidth from pinned memory (the e2e path's floor)."""
import time

import torch

dev = torch.device("cuda:0")
for gb in (1, 4):
    n = gb << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"H2D {gb} GiB pinned: {n / dt / 1e9:.1f} GB/s")
    t0 = time.perf_counter()
    for _ in range(3):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"D2H {gb} GiB pinned: {n / dt / 1e9:.1f} GB/s")
