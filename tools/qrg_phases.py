"""Phase breakdown of the big-block QR kernel k_qr_blocked_g (block 0, cycles), from a
-DCORU_QR_PROFILE build of the library selected with CORU_LIB_VARIANT=qrprof (tooling):
one TSQR of an m x d sketch; prints cycles per phase summed over the tree's levels."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1810_07323_b200 as cg
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 110
    ctx = cg.Context(0)
    lib = cg.load_library()
    b = torch.randn(m, d, dtype=torch.float64, device="cuda")
    cg.tsqr(b, ctx=ctx)
    out = (C.c_longlong * 12)()
    lib.coru_debug_qrg_phases(out, 1)
    cg.tsqr(b, ctx=ctx)
    torch.cuda.synchronize()
    lib.coru_debug_qrg_phases(out, 1)
    names = ["load", "panel chain", "gram VtV", "larft", "Y = Vt C", "Z = T Y", "C -= V Z", "export"]
    tot = sum(out[i] for i in range(8))
    for i, n in enumerate(names):
        print(f"{n:12s} {out[i]:10d} cycles  {100.0 * out[i] / max(tot, 1):5.1f} %")
    print(f"total {tot} cycles over the tree's levels (block 0 of each)")


if __name__ == "__main__":
    main()
