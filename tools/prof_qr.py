"""Drive the QR kernels alone (C2 shapes) for ncu: TSQR of 4000x60 and QRCP of 60x60."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1810_07323_b200 as cg

ctx = cg.Context(0)
b = torch.randn(4000, 60, dtype=torch.float64, device="cuda")
m = torch.randn(60, 60, dtype=torch.float64, device="cuda")
for _ in range(4):
    q, r = cg.tsqr(b, ctx=ctx)
    cg.qrcp(m, ctx=ctx)
torch.cuda.synchronize()
print("ok")
