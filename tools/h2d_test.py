"""Pinned host->device copy bandwidth vs size (tooling only)."""
import torch
s = torch.cuda.Stream()
for mb in (0.25, 1, 2, 8, 32, 128):
    n = int(mb * 2**20 // 8)
    x = torch.randn(n, dtype=torch.float64).pin_memory()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(5):
                y.copy_(x, non_blocking=True)
            e1.record(s)
        e1.synchronize()
    us = e0.elapsed_time(e1) / 5 * 1e3
    print(f"{mb:7.2f} MB pinned H2D: {us:8.1f} us  {mb * 2**20 / us / 1e3:6.1f} GB/s")
