"""cuBLAS DGEMM on the A-pass shapes (library reference point for the skinny GEMM)."""
import torch
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
for (m, n, d) in [(4000, 4000, 60), (4000, 4000, 64), (200000, 2000, 110), (32768, 32768, 220)]:
    a = torch.randn(m, n, dtype=torch.float64, device="cuda")
    x = torch.randn(n, d, dtype=torch.float64, device="cuda")
    y = torch.randn(m, d, dtype=torch.float64, device="cuda")
    ms = t(lambda: torch.mm(a, x)); ms2 = t(lambda: torch.mm(a.T, y))
    fl = 2.0 * m * n * d
    print(f"{m}x{n} d={d}: A·X {ms*1e3:.1f} us {fl/ms/1e9:.1f} TF | A^T·Y {ms2*1e3:.1f} us {fl/ms2/1e9:.1f} TF")
    del a
