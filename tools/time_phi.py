import time, sys
sys.path.insert(0, '.')
import paper_1810_07323_b200 as cg
for thr in (1, 4, 8, 16):
    t = time.perf_counter()
    for _ in range(5):
        cg.gaussian(4000, 60, cg.RngSeed(42, 1), threads=thr)
    print("phi 4000x60 threads", thr, (time.perf_counter() - t) / 5 * 1e3, "ms")
