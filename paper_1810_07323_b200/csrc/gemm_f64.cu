// FP64 skinny GEMM on the sm_100a FP64 tensor pipe (DMMA m16n8k8), stream-K scheduled.
//
// Replaces the reference's scalar i-k-j matmul (proj/include/coru/matrix.hpp:115-131) at its
// hot-path call sites: corutv.hpp:55 (c1 = a·c2), :57 (c2 = at·c1, with `at` never formed),
// :90 (Q1^T·A·Q2), :94 (U = Q1·Q). tcgen05 has no f64 kind, so FP64 tensor work on B200 is
// DMMA; tools/fp64_peak.cu measured DMMA and DFMA both at ~36.5-37 TFLOP/s per GPU.
//
// Shape: the output is Mo x N with N = the sketch width (<= 256): one CTA tile spans ALL of N
// (WN warps of 32 columns), so A is streamed from HBM exactly once per pass; warps own
// (16·MT) x 32 output tiles. K is the long dimension, staged in BK-deep slabs through an
// ST-deep cp.async ring in padded shared memory. A fragments are read as 16-byte pairs by giving
// lane t the k-pair (2t, 2t+1) instead of (t, t+4) (a consistent permutation of k in A and X, so
// the product is unchanged). A is streamed with an L2 evict-first policy so X stays L2-resident.
// Work is split stream-K style: P = resident CTAs, each owning an equal contiguous range of
// (tile, k-slab) iterations; tiles owned by one CTA are written directly. A split tile's segments
// are written to a workspace slot each and published with a release flag (tagged with a per-launch
// epoch); the CTA that owns the tile's LAST k-slab (the tile sits at the start of its range, so
// every other segment belongs to a lower-index, already-dispatched CTA: no deadlock) sums the
// segments in segment order after finishing its own range and writes C — the fix-up runs inside
// the GEMM (no second launch), in a fixed order (deterministic, no floating-point atomics).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

template <int WM_, int WN_, int MT_, int BK_, int ST_, bool TRANS_>
struct Cfg {
    static constexpr int WM = WM_, WN = WN_, MT = MT_, BK = BK_, ST = ST_;
    static constexpr bool TRANS = TRANS_;
    static constexpr int WTM = 16 * MT;  // warp tile rows
    static constexpr int BM = WM * WTM, BN = 32 * WN, NT = 32 * WM * WN;
    // op N: A tile [BM][BK+8]   (row stride = 8 mod 16 doubles: conflict-free 16-byte pair reads)
    // op T: A tile [BK][BM+4]   (row stride = 4 mod 16: 2 wavefronts per 8-byte fragment read)
    static constexpr int a_stride = TRANS ? BM + 4 : BK + 8;
    static constexpr int a_elems = TRANS ? BK * a_stride : BM * a_stride;
    static constexpr int x_stride = BN + 4;
    static constexpr int x_elems = BK * x_stride;
    static constexpr int stage_elems = a_elems + x_elems;
    static constexpr int bytes = ST * stage_elems * 8;
    static constexpr int regs = MT == 4 ? 192 : (MT == 2 ? 128 : 96);
    static constexpr int occ_smem = (227 * 1024) / bytes;
    static constexpr int occ_regs = 65536 / (NT * regs);
    static constexpr int min_blocks = occ_smem < occ_regs ? (occ_smem < 4 ? occ_smem : 4) : (occ_regs < 4 ? occ_regs : 4);
};

// Generic loader (any alignment; 8-byte copies when lda is odd).
template <class S, int VEC>
__device__ __forceinline__ void load_stage(double* sa, double* sx, const double* __restrict__ A, int64_t lda,
                                           const double* __restrict__ X, int64_t ldx, int64_t m0, int64_t k0,
                                           int64_t Mo, int64_t K, int N, int tid) {
    if constexpr (!S::TRANS) {
        constexpr int CPR = S::BK / VEC;
        for (int c = tid; c < S::BM * CPR; c += S::NT) {
            const int r = c / CPR, cc = (c % CPR) * VEC;
            const int64_t gr = m0 + r, gc = k0 + cc;
            int bytes = 0;
            const double* src = A;
            if (gr < Mo && gc < K) {
                bytes = int(imin64(VEC, K - gc)) * 8;
                src = A + gr * lda + gc;
            }
            cp_async_zfill<VEC * 8>(sa + r * S::a_stride + cc, src, bytes);
        }
    } else {
        constexpr int CPR = S::BM / VEC;
        for (int c = tid; c < S::BK * CPR; c += S::NT) {
            const int r = c / CPR, cc = (c % CPR) * VEC;
            const int64_t gr = k0 + r, gc = m0 + cc;
            int bytes = 0;
            const double* src = A;
            if (gr < K && gc < Mo) {
                bytes = int(imin64(VEC, Mo - gc)) * 8;
                src = A + gr * lda + gc;
            }
            cp_async_zfill<VEC * 8>(sa + r * S::a_stride + cc, src, bytes);
        }
    }
    constexpr int CPRX = S::BN / 2;  // X rows are 16-B aligned (ldx even, base aligned)
    for (int c = tid; c < S::BK * CPRX; c += S::NT) {
        const int r = c / CPRX, cc = (c % CPRX) * 2;
        const int64_t gr = k0 + r;
        int bytes = 0;
        const double* src = X;
        if (gr < K && cc < N) {
            bytes = int(imin64(2, N - cc)) * 8;
            src = X + gr * ldx + cc;
        }
        cp_async_zfill<16>(sx + r * S::x_stride + cc, src, bytes);
    }
}

// Loader for 16-byte-aligned operands: every thread's chunk columns and row offsets are fixed
// per tile, so a stage costs one pointer bump + one predicate per 16-byte copy.
template <class S>
struct FastLoader {
    static constexpr int A_CPR = S::TRANS ? S::BM / 2 : S::BK / 2;  // 16-byte chunks per smem row
    static constexpr int A_ROWS = S::TRANS ? S::BK : S::BM;
    static constexpr int A_RPP = S::NT / A_CPR;  // rows per pass
    static constexpr int A_PASSES = (A_ROWS + A_RPP - 1) / A_RPP;
    static constexpr int X_CPR = S::BN / 2;
    static constexpr int X_RPP = S::NT / X_CPR;
    static constexpr int X_PASSES = (S::BK + X_RPP - 1) / X_RPP;
    static_assert(S::NT % A_CPR == 0 && S::NT % X_CPR == 0, "thread mapping");
    static_assert(A_PASSES <= 32, "pass mask");

    const double* a_ptr;
    const double* x_ptr;
    int64_t a_pass_stride, a_k_stride, x_pass_stride;
    int a_r0, a_cc, x_r0, x_cc;
    int a_fixed_bytes;  // op T: bytes valid along m (fixed per tile)
    uint32_t a_row_ok;  // pass i row inside the tile (and < Mo for op N)
    int x_bytes;
    int64_t K;
    uint64_t pol_a, pol_x;

    __device__ FastLoader(const double* A, int64_t lda, const double* X, int64_t ldx, int64_t m0, int64_t Mo,
                          int64_t K_, int N, int tid, uint64_t pa, uint64_t px)  // X, N: this n-tile's columns
        : K(K_), pol_a(pa), pol_x(px) {
        a_r0 = tid / A_CPR;
        a_cc = (tid % A_CPR) * 2;
        x_r0 = tid / X_CPR;
        x_cc = (tid % X_CPR) * 2;
        a_row_ok = 0;
        if constexpr (!S::TRANS) {
            a_ptr = A + (m0 + a_r0) * lda + a_cc;
            a_pass_stride = int64_t(A_RPP) * lda;
            a_k_stride = 1;
#pragma unroll
            for (int i = 0; i < A_PASSES; ++i)
                if (a_r0 + i * A_RPP < A_ROWS && m0 + a_r0 + i * A_RPP < Mo) a_row_ok |= 1u << i;
            a_fixed_bytes = 16;
        } else {
            a_ptr = A + int64_t(a_r0) * lda + m0 + a_cc;
            a_pass_stride = int64_t(A_RPP) * lda;
            a_k_stride = lda;
#pragma unroll
            for (int i = 0; i < A_PASSES; ++i)
                if (a_r0 + i * A_RPP < A_ROWS) a_row_ok |= 1u << i;
            const int64_t rem = Mo - (m0 + a_cc);
            a_fixed_bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
        }
        x_ptr = X + int64_t(x_r0) * ldx + x_cc;
        x_pass_stride = int64_t(X_RPP) * ldx;
        x_bytes = N - x_cc >= 2 ? 16 : (N - x_cc == 1 ? 8 : 0);
    }

    __device__ __forceinline__ void load(double* sa, double* sx, int64_t k0, const double* A, const double* X,
                                         int64_t ldx) const {
        if constexpr (!S::TRANS) {
            const int64_t kr = K - (k0 + a_cc);
            const int kbytes = kr >= 2 ? 16 : (kr == 1 ? 8 : 0);
#pragma unroll
            for (int i = 0; i < A_PASSES; ++i) {
                if (a_r0 + i * A_RPP >= A_ROWS) continue;
                const bool ok = ((a_row_ok >> i) & 1u) && kbytes > 0;
                cp_async16_hint(sa + (a_r0 + i * A_RPP) * S::a_stride + a_cc, ok ? a_ptr + i * a_pass_stride + k0 : A,
                                ok ? kbytes : 0, pol_a);
            }
        } else {
#pragma unroll
            for (int i = 0; i < A_PASSES; ++i) {
                if (a_r0 + i * A_RPP >= A_ROWS) continue;
                const bool ok = k0 + a_r0 + i * A_RPP < K && a_fixed_bytes > 0;
                cp_async16_hint(sa + (a_r0 + i * A_RPP) * S::a_stride + a_cc,
                                ok ? a_ptr + i * a_pass_stride + k0 * a_k_stride : A, ok ? a_fixed_bytes : 0, pol_a);
            }
        }
#pragma unroll
        for (int i = 0; i < X_PASSES; ++i) {
            if (x_r0 + i * X_RPP >= S::BK) continue;
            const bool ok = k0 + x_r0 + i * X_RPP < K && x_bytes > 0;
            cp_async16_hint(sx + (x_r0 + i * X_RPP) * S::x_stride + x_cc, ok ? x_ptr + i * x_pass_stride + k0 * ldx : X,
                            ok ? x_bytes : 0, pol_x);
        }
    }
};

__device__ __forceinline__ void st_release_gpu_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// CTA c owns iterations [I*c/P, I*(c+1)/P) of the (tile, k-slab) space, tile-major.
__host__ __device__ __forceinline__ int64_t sk_begin(int64_t iters, int P, int c) { return iters * c / P; }
// The CTA that owns iteration g.
__host__ __device__ __forceinline__ int sk_owner(int64_t iters, int P, int64_t g) {
    return int(((g + 1) * P - 1) / iters);
}

template <class S, int VEC>
__global__ void __launch_bounds__(S::NT, S::min_blocks)
    k_gemm_f64(const double* __restrict__ A, int64_t lda, const double* __restrict__ X, int64_t ldx,
               double* __restrict__ C, int64_t ldc, int64_t Mo, int64_t K, int N, int64_t ktiles, int64_t iters, int P,
               double* __restrict__ ws, int max_seg, uint64_t* __restrict__ flags, uint64_t epoch, int G, int apol) {
    constexpr int MT = S::MT, BK = S::BK, ST = S::ST;
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / S::WN) * S::WTM, wn0 = (warp % S::WN) * 32;
    // Grouped stream-K: G = n-tiles groups of P CTAs each; group g owns n-tile g of every row block
    // and splits its (row block, k-slab) iterations stream-K style over its P CTAs. CTAs of equal
    // rank in different groups walk the same A rows at the same time, so A comes from DRAM once
    // and the other n-tiles read it from L2 (iters, P and `cta` below are per group).
    const int grp = int(blockIdx.x) % G;
    const int cta = int(blockIdx.x) / G;
    int64_t it = sk_begin(iters, P, cta);
    const int64_t it_end = sk_begin(iters, P, cta + 1);
    // A: evict-first when one CTA is its only reader; with n-tile groups every A line has G readers
    // within a short window, so it keeps the normal priority (apol: tooling override, -1 = auto).
    const int ap = apol >= 0 ? apol : (G > 1 ? 1 : 0);
    const uint64_t pol_a = ap == 0 ? l2_policy_evict_first() : (ap == 1 ? l2_policy_evict_normal() : l2_policy_evict_last());
    const uint64_t pol_x = l2_policy_evict_last();

    const int tiles_n = (N + S::BN - 1) / S::BN;
    int64_t fix_tile = -1;  // split tile whose last k-slab this CTA owns: summed after the range
    int fix_segs = 0;
    while (it < it_end) {
        const int64_t tile_m = it / ktiles;          // row block within the group
        const int64_t tile = G > 1 ? tile_m * tiles_n + grp : tile_m;  // global tile id (ws / flags)
        const int64_t kb = it % ktiles;
        const int64_t ke = imin64(ktiles, kb + (it_end - it));
        const int nk = int(ke - kb);
        const int64_t m0 = (G > 1 ? tile_m : tile / tiles_n) * S::BM;  // G == 1: n-tiles of a row block adjacent
        const int n0 = (G > 1 ? grp : int(tile % tiles_n)) * S::BN;
        const int Nt = N - n0;                        // columns left from this n-tile
        const double* Xt = X + n0;

        double acc[MT][4][4];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

        const FastLoader<S> fl(A, lda, Xt, ldx, m0, Mo, K, Nt, tid, pol_a, pol_x);
        auto stage_load = [&](double* sa, int64_t k0) {
            if constexpr (VEC == 2) fl.load(sa, sa + S::a_elems, k0, A, Xt, ldx);
            else load_stage<S, VEC>(sa, sa + S::a_elems, A, lda, Xt, ldx, m0, k0, Mo, K, Nt, tid);
        };
        __syncthreads();  // previous segment's readers are done with the ring
#pragma unroll
        for (int s = 0; s < ST - 1; ++s) {
            if (s < nk) stage_load(smem + s * S::stage_elems, (kb + s) * BK);
            cp_async_commit();
        }
        for (int ki = 0; ki < nk; ++ki) {
            cp_async_wait<ST - 2>();
            __syncthreads();
            {
                const int nxt = ki + ST - 1;
                if (nxt < nk) stage_load(smem + (nxt % ST) * S::stage_elems, (kb + nxt) * BK);
                cp_async_commit();
            }
            const double* sa = smem + (ki % ST) * S::stage_elems;
            const double* sx = sa + S::a_elems;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 8) {
                // lane (g, t) holds k-pair (2t, 2t+1) of the k8 slab for both operands
                double af[MT][4], bf[4][2];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int r = wm0 + mt * 16 + g;
                    if constexpr (!S::TRANS) {
                        const double2 lo = *reinterpret_cast<const double2*>(sa + r * S::a_stride + kk + 2 * t);
                        const double2 hi = *reinterpret_cast<const double2*>(sa + (r + 8) * S::a_stride + kk + 2 * t);
                        af[mt][0] = lo.x;
                        af[mt][2] = lo.y;
                        af[mt][1] = hi.x;
                        af[mt][3] = hi.y;
                    } else {
                        af[mt][0] = sa[(kk + 2 * t) * S::a_stride + r];
                        af[mt][1] = sa[(kk + 2 * t) * S::a_stride + r + 8];
                        af[mt][2] = sa[(kk + 2 * t + 1) * S::a_stride + r];
                        af[mt][3] = sa[(kk + 2 * t + 1) * S::a_stride + r + 8];
                    }
                }
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const int c = wn0 + nt * 8 + g;
                    bf[nt][0] = sx[(kk + 2 * t) * S::x_stride + c];
                    bf[nt][1] = sx[(kk + 2 * t + 1) * S::x_stride + c];
                }
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma_16x8x8(acc[mt][nt], af[mt], bf[nt]);
            }
        }
        cp_async_wait<0>();

        // Epilogue: whole tile owned -> C; otherwise -> this segment's slot of the tile.
        const bool whole = kb == 0 && ke == ktiles;
        double* dst_base;
        int64_t ld_dst, row_base;
        int seg = 0;
        if (whole) {
            dst_base = C + n0;
            ld_dst = ldc;
            row_base = m0;
        } else {
            const int first = sk_owner(iters, P, tile_m * ktiles);
            seg = cta - first;
            dst_base = ws + (tile * max_seg + seg) * int64_t(S::BM * S::BN);
            ld_dst = S::BN;
            row_base = 0;
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = wm0 + mt * 16 + g + h * 8;
                if (m0 + r >= Mo) continue;
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const int col = wn0 + nt * 8 + 2 * t;
                    double* dst = dst_base + (row_base + r) * ld_dst + col;
                    if (!whole) {
                        *reinterpret_cast<double2*>(dst) = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
                    } else if (col + 1 < Nt && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                        *reinterpret_cast<double2*>(dst) = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
                    } else if (col < Nt) {
                        dst[0] = acc[mt][nt][2 * h];
                        if (col + 1 < Nt) dst[1] = acc[mt][nt][2 * h + 1];
                    }
                }
            }
        }
        if (!whole) {
            if (ke == ktiles) {  // last segment: this CTA sums the tile once its range is done
                fix_tile = tile;
                fix_segs = seg + 1;
            } else {             // publish the segment
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    st_release_gpu_u64(flags + tile * max_seg + seg, epoch);
                }
            }
        }
        it = tile_m * ktiles + ke;
    }
    if (fix_tile >= 0) {
        // Fixed-order sum of the tile's segments (seg 0 .. fix_segs-1; the last one is ours).
        if (tid == 0) {
            for (int q = 0; q + 1 < fix_segs; ++q) {
                const uint64_t* f = flags + fix_tile * max_seg + q;
                if (ld_acquire_gpu_u64(f) != epoch) {
                    const long long t0 = clock64();
                    while (ld_acquire_gpu_u64(f) != epoch)
                        if (clock64() - t0 > 16000000000LL) __trap();  // never hang the GPU
                }
            }
        }
        __syncthreads();
        const int64_t m0 = (fix_tile / tiles_n) * S::BM;
        const int n0 = int(fix_tile % tiles_n) * S::BN;
        constexpr int TE2 = S::BM * S::BN / 2, VPT = 4;  // double2 elements; 4 per thread in flight
        const int64_t te = int64_t(S::BM) * S::BN;
        const double2* base = reinterpret_cast<const double2*>(ws + fix_tile * max_seg * te);
        for (int e0 = tid; e0 < TE2; e0 += S::NT * VPT) {
            double2 acc[VPT];
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const int e2 = e0 + v * S::NT;
                acc[v] = e2 < TE2 ? __ldcg(base + e2) : make_double2(0.0, 0.0);
            }
#pragma unroll 4
            for (int q = 1; q < fix_segs; ++q) {
                double2 t[VPT];
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    const int e2 = e0 + v * S::NT;
                    t[v] = e2 < TE2 ? __ldcg(base + q * (te / 2) + e2) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int v = 0; v < VPT; ++v) { acc[v].x += t[v].x; acc[v].y += t[v].y; }
            }
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                const int e2 = e0 + v * S::NT;
                if (e2 >= TE2) continue;
                const int r = (2 * e2) / S::BN, cc = (2 * e2) % S::BN;
                if (m0 + r >= Mo) continue;
                double* dst = C + (m0 + r) * ldc + n0 + cc;
                if (n0 + cc < N) dst[0] = acc[v].x;
                if (n0 + cc + 1 < N) dst[1] = acc[v].y;
            }
        }
        // The consumer clears the flags it waited on: a CUDA-graph replay of this launch carries the
        // same epoch, and must not take the previous replay's publishes for its own.
        if (tid == 0)
            for (int q = 0; q + 1 < fix_segs; ++q) flags[fix_tile * max_seg + q] = 0;
    }
}

// ---- configuration table -------------------------------------------------------------------
struct CfgInfo {
    int id, wm, wn, mt, bk, st;
};
// Candidates per sketch-width class (WN = ceil(N/32)); tools/gemm_tune.cu sweeps them.
#define CORU_GEMM_CONFIGS(X) \
    X(0, 4, 1, 2, 16, 3)     \
    X(1, 4, 2, 2, 16, 3)     \
    X(2, 4, 2, 4, 16, 3)     \
    X(3, 2, 2, 4, 32, 3)     \
    X(4, 2, 3, 2, 16, 3)     \
    X(5, 2, 4, 2, 16, 3)     \
    X(6, 2, 4, 4, 16, 3)     \
    X(7, 1, 5, 2, 16, 3)     \
    X(8, 1, 6, 2, 16, 3)     \
    X(9, 1, 7, 2, 16, 3)     \
    X(10, 1, 7, 4, 16, 3)    \
    X(11, 1, 8, 2, 16, 2)    \
    X(12, 1, 8, 4, 16, 2)    \
    X(13, 4, 2, 2, 32, 3)    \
    X(14, 1, 7, 4, 32, 2)    \
    X(15, 2, 1, 2, 16, 4)    \
    X(16, 2, 2, 1, 16, 4)    \
    X(17, 2, 2, 2, 16, 3)    \
    X(18, 4, 1, 1, 16, 4)    \
    X(19, 1, 2, 2, 16, 4)

constexpr CfgInfo kCfgs[] = {
#define CORU_ROW(id, wm, wn, mt, bk, st) {id, wm, wn, mt, bk, st},
    CORU_GEMM_CONFIGS(CORU_ROW)
#undef CORU_ROW
};
constexpr int kNumCfgs = int(sizeof(kCfgs) / sizeof(kCfgs[0]));

int cfg_bytes(const CfgInfo& c, bool trans) {
    const int bm = c.wm * 16 * c.mt, bn = 32 * c.wn;
    const int a = trans ? c.bk * (bm + 4) : bm * (c.bk + 8);
    return c.st * (a + c.bk * (bn + 4)) * 8;
}

// Picked from tools/gemm_tune.cu on B200 (round 1): small 4-warp CTAs with 4-deep rings and 32- or
// 64-wide n-tiles (3-4 resident CTAs per SM, A re-read from L2 per n-tile) beat the wide-tile
// variants by 10-15 % on every BASELINE shape.
int default_cfg(Op op, int N) {
    if (op == Op::N) return N <= 32 ? 0 : (N <= 64 ? 16 : 0);
    return N <= 32 ? 15 : (N <= 64 ? 19 : 15);
}

// Fix-up flag epochs: ONE process-wide counter for every configuration. (Per-configuration
// counters let two GEMMs of different configurations that reuse a workspace carry the same epoch,
// so a stale flag of the earlier one could pass for a fresh publish of the later one.)
std::atomic<uint64_t> g_gemm_epoch{0};

// Tooling knob (tests/test_gpu_kernels.py planner sweep): at most this many CTAs per output tile
// (0 = the planner's own choice). Read by every plan, so workspace sizes stay consistent.
std::atomic<int> g_gemm_split_cap{0};

template <class S>
cudaError_t launch_cfg(const double* A, int64_t lda, const double* X, int64_t ldx, double* C, int64_t ldc, int64_t Mo,
                       int64_t K, int N, const GemmPlan& p, double* ws, cudaStream_t st) {
    const int64_t ktiles = (K + S::BK - 1) / S::BK;
    const int64_t tiles = ((Mo + S::BM - 1) / S::BM) * ((N + S::BN - 1) / S::BN);
    const int G = p.groups;
    static const int apol = getenv("CORU_GEMM_APOL") ? atoi(getenv("CORU_GEMM_APOL")) : -1;
    const int64_t iters = (G > 1 ? (Mo + S::BM - 1) / S::BM : tiles) * ktiles;  // per group
    const bool vec = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
    // split-tile flags live after the partial tiles; a fresh epoch per launch (no reset needed)
    uint64_t* flags = p.fixup ? reinterpret_cast<uint64_t*>(ws + tiles * int64_t(p.max_seg) * S::BM * S::BN) : nullptr;
    const uint64_t epoch = 0xC0DEull << 48 | (++g_gemm_epoch & 0xFFFFFFFFFFFFull);
    if (vec) {
        auto k = k_gemm_f64<S, 2>;
        allow_max_smem(k);
        k<<<p.splits * G, S::NT, S::bytes, st>>>(A, lda, X, ldx, C, ldc, Mo, K, N, ktiles, iters, p.splits, ws,
                                                  p.max_seg, flags, epoch, G, apol);
    } else {
        auto k = k_gemm_f64<S, 1>;
        allow_max_smem(k);
        k<<<p.splits * G, S::NT, S::bytes, st>>>(A, lda, X, ldx, C, ldc, Mo, K, N, ktiles, iters, p.splits, ws,
                                                  p.max_seg, flags, epoch, G, apol);
    }
    return cudaGetLastError();
}

}  // namespace

int gemm_f64_num_configs() { return kNumCfgs; }
void gemm_f64_set_split_cap(int cap) { g_gemm_split_cap.store(cap < 0 ? 0 : cap); }

GemmPlan plan_gemm_f64_cfg(Op op, int64_t Mo, int64_t K, int N, int num_sms, int cfg) {
    GemmPlan p;
    if (cfg < 0 || cfg >= kNumCfgs) cfg = default_cfg(op, N);
    const CfgInfo& c = kCfgs[cfg];
    p.cfg = cfg;
    p.bm = c.wm * 16 * c.mt;
    p.bn = 32 * c.wn;
    const int64_t ktiles = (K + c.bk - 1) / c.bk;
    const int64_t tiles_m = (Mo + p.bm - 1) / p.bm, tiles_n = (N + p.bn - 1) / p.bn;
    const int64_t tiles = tiles_m * tiles_n;
    const int nt = 32 * c.wm * c.wn;
    const int reg_per_thread = c.mt == 4 ? 192 : (c.mt == 2 ? 128 : 96);
    const int occ_smem = (227 * 1024) / cfg_bytes(c, op == Op::T);
    const int occ_regs = 65536 / (nt * reg_per_thread);
    const int occ = std::max(1, std::min({4, occ_smem, occ_regs}));
    // Every CTA resident at once, each owns >= 4 k-slabs, and no tile is shared by more CTAs than
    // needed to fill the machine (bounded fix-up).
    // Grouped stream-K (several n-tiles): one CTA group per n-tile walking the row blocks in step,
    // so A is read from DRAM once per pass instead of once per n-tile (k_gemm_f64).
    static const bool grouped_env = getenv("CORU_GEMM_GROUPED") == nullptr || atoi(getenv("CORU_GEMM_GROUPED")) != 0;
    const int64_t resident = int64_t(occ) * num_sms;
    const int G = (grouped_env && tiles_n > 1 && resident / tiles_n >= 8) ? int(tiles_n) : 1;
    p.groups = G;
    const int64_t gtiles = G > 1 ? tiles_m : tiles;  // tiles per group
    const int64_t iters = gtiles * ktiles;            // iterations per group
    int64_t P64 = std::min<int64_t>(resident / G, iters / 4);
    P64 = std::min<int64_t>(P64, gtiles * std::max<int64_t>(12, (resident / G + gtiles - 1) / gtiles));
    if (const int cap = g_gemm_split_cap.load(std::memory_order_relaxed); cap > 0)
        P64 = std::min<int64_t>(P64, gtiles * cap);
    const int P = int(std::max<int64_t>(P64, 1));     // CTAs per group
    p.splits = P;
    const int64_t per = std::max<int64_t>(1, iters / P);
    p.max_seg = int(std::min<int64_t>(P, (ktiles + per - 1) / per + 1));
    p.fixup = false;
    for (int64_t tile = 0; tile < gtiles && !p.fixup; ++tile) {
        const int64_t g0 = tile * ktiles, g1 = g0 + ktiles - 1;
        p.fixup = ((g0 + 1) * P - 1) / iters != ((g1 + 1) * P - 1) / iters;
    }
    p.ws_elems = p.fixup ? tiles * int64_t(p.max_seg) * (int64_t(p.bm) * p.bn + 1) : 0;  // partials + flags
    p.num_sms = num_sms;
    return p;
}

GemmPlan plan_gemm_f64(Op op, int64_t Mo, int64_t K, int N, int num_sms) {
    // Sketch widths beyond one CTA tile run as 256-wide column chunks (see gemm_f64); the
    // workspace covers the largest chunk plan.
    GemmPlan p = plan_gemm_f64_cfg(op, Mo, K, std::min(N, 256), num_sms, -1);
    for (int n0 = 256; n0 < N; n0 += 256)
        p.ws_elems = std::max(p.ws_elems, plan_gemm_f64_cfg(op, Mo, K, std::min(256, N - n0), num_sms, -1).ws_elems);
    return p;
}

cudaError_t gemm_f64(Op op, const double* A, int64_t lda, const double* X, int64_t ldx, double* C, int64_t ldc,
                     int64_t Mo, int64_t K, int N, const GemmPlan& p, double* ws, cudaStream_t st) {
    if (Mo <= 0 || N <= 0) return cudaSuccess;
    if (N > 256) {  // independent column chunks of X and C (plans are built for <= 256 columns)
        for (int n0 = 0; n0 < N; n0 += 256) {
            const int nc = std::min(256, N - n0);
            const GemmPlan q = plan_gemm_f64_cfg(op, Mo, K, nc, p.num_sms, -1);
            cudaError_t e = gemm_f64(op, A, lda, X + n0, ldx, C + n0, ldc, Mo, K, nc, q, ws, st);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
#define CORU_CASE(id, wm, wn, mt, bk, st_)                                                                   \
    if (p.cfg == id)                                                                                           \
        return op == Op::N                                                                                     \
                   ? launch_cfg<Cfg<wm, wn, mt, bk, st_, false>>(A, lda, X, ldx, C, ldc, Mo, K, N, p, ws, st)  \
                   : launch_cfg<Cfg<wm, wn, mt, bk, st_, true>>(A, lda, X, ldx, C, ldc, Mo, K, N, p, ws, st);
    CORU_GEMM_CONFIGS(CORU_CASE)
#undef CORU_CASE
    return cudaErrorInvalidValue;
}

}  // namespace coru_gpu
