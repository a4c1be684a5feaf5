"""Per-stage cost vs. per-CTA overhead of the int8 A-pass kernels (tooling): op-N products of a
200000-row A at K = 1024 / 2048 / 4096 and several sketch widths; the A-pass time is read from the
context's own CUDA events (coru_ctx_profile_apass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1810_07323_b200 as cg
    ctx = cg.Context(0)
    m = int(os.environ.get("M", 200000))
    g = torch.Generator(device="cuda").manual_seed(1)
    for eng, name in ((2, "inline"), (3, "planes")):
        ctx.set_f64_engine(eng)
        for n in (64, 112, 128):
            res = []
            for k in (1024, 2048, 4096):
                a = torch.randn((m, k), dtype=torch.float64, device="cuda", generator=g)
                x = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g)
                for _ in range(2):
                    cg.gemm(a, x, op=0, ctx=ctx)
                ctx.set_profiling(True)
                ctx.profile_apass()
                reps = 5
                for _ in range(reps):
                    cg.gemm(a, x, op=0, ctx=ctx)
                p = ctx.profile_apass()
                ctx.set_profiling(False)
                res.append(p["ms"] / reps)
                del a, x
            slope = (res[2] - res[1]) / 2048 * 1000   # us per k over all CTAs
            icpt = res[1] - slope * 2048 / 1000
            print(f"{name} N={n}: K=1024 {res[0]:.3f} ms, 2048 {res[1]:.3f} ms, 4096 {res[2]:.3f} ms; "
                  f"marginal {slope * 2000 / 1000:.3f} ms per 2000 k, intercept {icpt:.3f} ms", flush=True)
    ctx.set_f64_engine(ctx.F64_AUTO)


if __name__ == "__main__":
    main()
