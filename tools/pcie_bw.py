"""H2D / D2H bandwidth on this box: contiguous pinned copies and the 2-D
pattern the one-shot call's column groups use (16 KB rows, N*8-byte pitch)."""
import time

import torch

n = 32400
dev = torch.empty((n, 2048), dtype=torch.float64, device="cuda")
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
flat = torch.empty(n * 2048, dtype=torch.float64, pin_memory=True)
for name, fn, nbytes in [
    ("D2H contiguous", lambda: flat.copy_(dev.view(-1), non_blocking=True), dev.numel() * 8),
    ("H2D contiguous", lambda: dev.view(-1).copy_(flat, non_blocking=True), dev.numel() * 8),
    ("D2H 2-D (16 KB rows, pitched)", lambda: host[:, :2048].copy_(dev, non_blocking=True), dev.numel() * 8),
]:
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s")
