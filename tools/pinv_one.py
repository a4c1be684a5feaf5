import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1810_07323_b200 as cg
ctx = cg.Context(0)
rng = np.random.default_rng(60)
a = rng.standard_normal((60, 60)) * (0.75 ** np.arange(60))
ad = torch.from_numpy(a).cuda()
for _ in range(2): cg.pinv(ad, ctx=ctx)
torch.cuda.synchronize()
