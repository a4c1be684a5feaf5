"""Device vs host Φ generator: ulp statistics and the worst entries (tooling)."""
import sys; sys.path.insert(0, ".")
import numpy as np, paper_1810_07323_b200 as cg
from oracle import Oracle
o = Oracle()
ctx = cg.Context(0)
for rows, cols, ld, seed, stream in [(7, 9, 9, 42, 3), (1, 5, 8, 7, 0), (4001, 61, 64, 5, 2), (100, 100, 100, 42, 0), (65536, 520, 520, 42, 7)]:
    g = cg.gaussian_device(rows, cols, cg.RngSeed(seed, stream), ctx=ctx, ld=ld).cpu().numpy()[:, :cols]
    h = cg.gaussian(rows, cols, cg.RngSeed(seed, stream), threads=16)
    gi, hi = g.view(np.int64) if g.flags.c_contiguous else np.ascontiguousarray(g).view(np.int64), h.view(np.int64)
    u = np.abs(gi - hi)
    i = np.unravel_index(np.argmax(u), u.shape)
    print(rows, cols, "max int-ulp", u.max(), "at", i, "g", repr(g[i]), "h", repr(h[i]), "n>4", int(np.sum(u > 4)))
    if u.max() > 4 and rows * cols < 40_000_000:
        ho = o.gaussian(rows, cols, seed, stream)
        print("   host==oracle:", np.array_equal(h, ho), " oracle at i:", repr(ho[i]), " rows bad:", np.unique(np.argwhere(u > 4)[:, 0])[:10])
