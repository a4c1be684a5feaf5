import torch, time
x = torch.empty(4000 * 64, dtype=torch.float64).pin_memory()
y = torch.empty(4000 * 64, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
for n in (1, 2, 5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(n):
            y.copy_(x, non_blocking=True)
        e1.record(s)
    e1.synchronize()
    print(f"{n} x 2 MB pinned H2D: {e0.elapsed_time(e1) / n * 1e3:.1f} us each")
