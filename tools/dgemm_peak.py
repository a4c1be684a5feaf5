"""Measure cuBLAS DGEMM (fp64) throughput on this GPU: the FP64 roofline denominator.

MEASURED_PEAKS.json carries only HBM and bf16 peaks; the fp64 A-passes of CoR-UTV are
FP64-compute-bound, so the FP64 peak is measured here the same way the
driver measures bf16 (torch.matmul -> cuBLAS, best of N with CUDA events).
"""
import json, sys, time
import torch


def dgemm_tflops(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    print(json.dumps({"dgemm_tflops": dgemm_tflops(n), "n": n}))
