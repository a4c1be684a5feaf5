// FP64 skinny GEMM on the sm_100a FP64 tensor pipe (DMMA m16n8k8), stream-K scheduled.
//
// Replaces the reference's scalar i-k-j matmul (proj/include/coru/matrix.hpp:115-131) at its
// hot-path call sites: corutv.hpp:55 (c1 = a·c2), :57 (c2 = at·c1, with `at` never formed),
// :90 (Q1^T·A·Q2), :94 (U = Q1·Q). tcgen05 has no f64 kind, so FP64 tensor work on B200 is
// DMMA; tools/fp64_peak.cu measured DMMA and DFMA both at ~36.5-37 TFLOP/s per GPU.
//
// Shape: the output is Mo x N with N = the sketch width (<= 256): one CTA tile spans ALL of N
// (warps 32x32, WN = ceil(N/32) warps across, WM = 8/WN down), so A is streamed from HBM exactly
// once per pass. K is the long dimension. BK = 16 slabs go through a 3-deep cp.async ring in
// padded shared memory; A fragments are read as 16-byte pairs by giving each lane the k-pair
// (2t, 2t+1) instead of (t, t+4) (a consistent permutation of k in A and X, so the product is
// unchanged). Work is split stream-K style: exactly P = 2 x SMs CTAs, each owning an equal
// contiguous range of (tile, k-slab) iterations; tiles owned by one CTA are written directly,
// split tiles go through a fixed-order fix-up (deterministic, no atomics).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kBK = 16;
constexpr int kStages = 3;

template <int WM, int WN, bool TRANS>
struct Cfg {
    static constexpr int BM = 32 * WM, BN = 32 * WN, NT = 32 * WM * WN;
    // op N: A tile [BM][BK+8]   (row stride = 8 mod 16 doubles: conflict-free 16-byte pair reads)
    // op T: A tile [BK][BM+4]   (row stride = 4 mod 16: 2 wavefronts per 8-byte fragment read)
    static constexpr int a_stride = TRANS ? BM + 4 : kBK + 8;
    static constexpr int a_elems = TRANS ? kBK * a_stride : BM * a_stride;
    static constexpr int x_stride = BN + 4;
    static constexpr int x_elems = kBK * x_stride;
    static constexpr int stage_elems = a_elems + x_elems;
    static constexpr int bytes = kStages * stage_elems * 8;
};

template <int WM, int WN, bool TRANS, int VEC>
__device__ __forceinline__ void load_stage(double* sa, double* sx, const double* __restrict__ A, int64_t lda,
                                           const double* __restrict__ X, int64_t ldx, int64_t m0, int64_t k0,
                                           int64_t Mo, int64_t K, int N, int tid) {
    using S = Cfg<WM, WN, TRANS>;
    if constexpr (!TRANS) {
        constexpr int CPR = kBK / VEC;
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
        for (int c = tid; c < kBK * CPR; c += S::NT) {
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
    for (int c = tid; c < kBK * CPRX; c += S::NT) {
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

// CTA c owns iterations [I*c/P, I*(c+1)/P) of the (tile, k-slab) space, tile-major.
__host__ __device__ __forceinline__ int64_t sk_begin(int64_t iters, int P, int c) { return iters * c / P; }
// The CTA that owns iteration g.
__host__ __device__ __forceinline__ int sk_owner(int64_t iters, int P, int64_t g) {
    return int(((g + 1) * P - 1) / iters);
}

template <int WM, int WN, bool TRANS, int VEC>
__global__ void __launch_bounds__(32 * WM * WN, 2)
    k_gemm_f64(const double* __restrict__ A, int64_t lda, const double* __restrict__ X, int64_t ldx,
               double* __restrict__ C, int64_t ldc, int64_t Mo, int64_t K, int N, int64_t ktiles, int64_t iters, int P,
               double* __restrict__ ws, int max_seg) {
    using S = Cfg<WM, WN, TRANS>;
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / WN) * 32, wn0 = (warp % WN) * 32;
    const int cta = blockIdx.x;
    int64_t it = sk_begin(iters, P, cta);
    const int64_t it_end = sk_begin(iters, P, cta + 1);

    while (it < it_end) {
        const int64_t tile = it / ktiles;
        const int64_t kb = it % ktiles;
        const int64_t ke = imin64(ktiles, kb + (it_end - it));
        const int nk = int(ke - kb);
        const int64_t m0 = tile * S::BM;

        double acc[2][4][4];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

        __syncthreads();  // previous segment's readers are done with the ring
#pragma unroll
        for (int s = 0; s < kStages - 1; ++s) {
            if (s < nk) {
                double* sa = smem + s * S::stage_elems;
                load_stage<WM, WN, TRANS, VEC>(sa, sa + S::a_elems, A, lda, X, ldx, m0, (kb + s) * kBK, Mo, K, N, tid);
            }
            cp_async_commit();
        }
        for (int ki = 0; ki < nk; ++ki) {
            cp_async_wait<kStages - 2>();
            __syncthreads();
            {
                const int nxt = ki + kStages - 1;
                if (nxt < nk) {
                    double* sa = smem + (nxt % kStages) * S::stage_elems;
                    load_stage<WM, WN, TRANS, VEC>(sa, sa + S::a_elems, A, lda, X, ldx, m0, (kb + nxt) * kBK, Mo, K,
                                                   N, tid);
                }
                cp_async_commit();
            }
            const double* sa = smem + (ki % kStages) * S::stage_elems;
            const double* sx = sa + S::a_elems;
#pragma unroll
            for (int kk = 0; kk < kBK; kk += 8) {
                // lane (g, t) holds k-pair (2t, 2t+1) of the k8 slab for both operands
                double af[2][4], bf[4][2];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const int r = wm0 + mt * 16 + g;
                    if constexpr (!TRANS) {
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
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma_16x8x8(acc[mt][nt], af[mt], bf[nt]);
            }
        }
        cp_async_wait<0>();

        // Epilogue: whole tile owned -> C; otherwise -> this segment's slot of the tile.
        const bool whole = kb == 0 && ke == ktiles;
        double* dst_base;
        int64_t ld_dst, row_base;
        if (whole) {
            dst_base = C;
            ld_dst = ldc;
            row_base = m0;
        } else {
            const int first = sk_owner(iters, P, tile * ktiles);
            const int seg = cta - first;
            dst_base = ws + (tile * max_seg + seg) * int64_t(S::BM * S::BN);
            ld_dst = S::BN;
            row_base = 0;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
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
                    } else if (col + 1 < N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                        *reinterpret_cast<double2*>(dst) = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
                    } else if (col < N) {
                        dst[0] = acc[mt][nt][2 * h];
                        if (col + 1 < N) dst[1] = acc[mt][nt][2 * h + 1];
                    }
                }
            }
        }
        it = tile * ktiles + ke;
    }
}

// Fix-up of the split tiles: C(tile) = sum of its segments in CTA order (fixed order).
// grid = (tiles, element chunks of 256): every thread owns one element of one tile.
__global__ void k_streamk_fixup(const double* __restrict__ ws, int max_seg, int bm, int bn, int64_t ktiles,
                                int64_t iters, int P, double* __restrict__ C, int64_t ldc, int64_t Mo, int N) {
    const int64_t tile = blockIdx.x;
    const int first = sk_owner(iters, P, tile * ktiles);
    const int last = sk_owner(iters, P, tile * ktiles + ktiles - 1);
    if (first == last) return;  // written directly by its only owner
    const int64_t tile_elems = int64_t(bm) * bn;
    const int e = blockIdx.y * blockDim.x + threadIdx.x;
    if (e >= tile_elems) return;
    const int r = e / bn, c = e % bn;
    const int64_t row = tile * bm + r;
    if (row >= Mo || c >= N) return;
    const double* base = ws + tile * max_seg * tile_elems + e;
    double s = base[0];
    for (int q = 1; q <= last - first; ++q) s += base[q * tile_elems];
    C[row * ldc + c] = s;
}

void warp_grid(int N, int& wm, int& wn) {
    wn = std::max(1, std::min(8, (N + 31) / 32));
    wm = std::max(1, std::min(4, 8 / wn));
}

int cfg_bytes(int wm, int wn, bool trans) {
    const int bm = 32 * wm, bn = 32 * wn;
    const int a = trans ? kBK * (bm + 4) : bm * (kBK + 8);
    return kStages * (a + kBK * (bn + 4)) * 8;
}

template <int WM, int WN, bool TRANS>
cudaError_t launch(const double* A, int64_t lda, const double* X, int64_t ldx, double* C, int64_t ldc, int64_t Mo,
                   int64_t K, int N, const GemmPlan& p, double* ws, cudaStream_t st) {
    using S = Cfg<WM, WN, TRANS>;
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int64_t tiles = (Mo + S::BM - 1) / S::BM;
    const int64_t iters = tiles * ktiles;
    const bool vec = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
    if (vec) {
        auto k = k_gemm_f64<WM, WN, TRANS, 2>;
        allow_max_smem(k);
        k<<<p.splits, S::NT, S::bytes, st>>>(A, lda, X, ldx, C, ldc, Mo, K, N, ktiles, iters, p.splits, ws, p.max_seg);
    } else {
        auto k = k_gemm_f64<WM, WN, TRANS, 1>;
        allow_max_smem(k);
        k<<<p.splits, S::NT, S::bytes, st>>>(A, lda, X, ldx, C, ldc, Mo, K, N, ktiles, iters, p.splits, ws, p.max_seg);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !p.fixup) return e;
    const dim3 grid(unsigned(tiles), unsigned((S::BM * S::BN + 255) / 256));
    k_streamk_fixup<<<grid, 256, 0, st>>>(ws, p.max_seg, S::BM, S::BN, ktiles, iters, p.splits, C, ldc, Mo, N);
    return cudaGetLastError();
}

}  // namespace

GemmPlan plan_gemm_f64(Op op, int64_t Mo, int64_t K, int N, int num_sms) {
    (void)op;
    GemmPlan p;
    int wm, wn;
    warp_grid(N, wm, wn);
    p.bm = 32 * wm;
    p.bn = 32 * wn;
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int64_t tiles = (Mo + p.bm - 1) / p.bm;
    const int64_t iters = tiles * ktiles;
    // Every CTA resident at once (occupancy by shared memory), never more CTAs than iterations.
    const int occ = std::max(1, std::min(2, (227 * 1024) / cfg_bytes(wm, wn, op == Op::T)));
    // ... and each CTA owns >= 4 k-slabs, and no tile is shared by more than 12 CTAs (bounded fix-up).
    int64_t P64 = std::min<int64_t>(int64_t(occ) * num_sms, iters / 4);
    P64 = std::min<int64_t>(P64, tiles * 12);
    int P = int(std::max<int64_t>(P64, 1));
    p.splits = P;
    // Max segments a tile is split into: ceil(ktiles / (iters/P)) + 1.
    const int64_t per = std::max<int64_t>(1, iters / P);
    p.max_seg = int(std::min<int64_t>(P, (ktiles + per - 1) / per + 1));
    p.fixup = false;
    for (int64_t tile = 0; tile < tiles && !p.fixup; ++tile) {
        const int64_t g0 = tile * ktiles, g1 = g0 + ktiles - 1;
        p.fixup = ((g0 + 1) * P - 1) / iters != ((g1 + 1) * P - 1) / iters;
    }
    p.ws_elems = p.fixup ? tiles * int64_t(p.max_seg) * p.bm * p.bn : 0;
    return p;
}

cudaError_t gemm_f64(Op op, const double* A, int64_t lda, const double* X, int64_t ldx, double* C, int64_t ldc,
                     int64_t Mo, int64_t K, int N, const GemmPlan& p, double* ws, cudaStream_t st) {
    if (Mo <= 0 || N <= 0) return cudaSuccess;
    if (N > p.bn) {  // sketch widths beyond one CTA tile: independent column chunks of X and C
        for (int n0 = 0; n0 < N; n0 += p.bn) {
            const int nc = std::min(p.bn, N - n0);
            const GemmPlan q = plan_gemm_f64(op, Mo, K, nc, 148);
            cudaError_t e = gemm_f64(op, A, lda, X + n0, ldx, C + n0, ldc, Mo, K, nc, q, ws, st);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const int wn = p.bn / 32, wm = p.bm / 32;
#define CORU_CASE(WM_, WN_)                                                                   \
    if (wm == WM_ && wn == WN_)                                                               \
        return op == Op::N ? launch<WM_, WN_, false>(A, lda, X, ldx, C, ldc, Mo, K, N, p, ws, st) \
                           : launch<WM_, WN_, true>(A, lda, X, ldx, C, ldc, Mo, K, N, p, ws, st);
    CORU_CASE(4, 1)
    CORU_CASE(4, 2)
    CORU_CASE(2, 3)
    CORU_CASE(2, 4)
    CORU_CASE(1, 5)
    CORU_CASE(1, 6)
    CORU_CASE(1, 7)
    CORU_CASE(1, 8)
#undef CORU_CASE
    return cudaErrorInvalidValue;
}

}  // namespace coru_gpu
