import torch
m, n, d = 32768, 32768, 224
a = torch.randn(m, n, dtype=torch.float64, device="cuda")
x = torch.randn(n, d, dtype=torch.float64, device="cuda")
for _ in range(3): torch.mm(a, x)
torch.cuda.synchronize()
