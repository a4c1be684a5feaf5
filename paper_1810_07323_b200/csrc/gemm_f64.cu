// FP64 skinny GEMM on the sm_100a FP64 tensor pipe (DMMA m16n8k8).
//
// Replaces the reference's scalar i-k-j matmul (proj/include/coru/matrix.hpp:115-131) at its
// hot-path call sites: corutv.hpp:55 (c1 = a·c2), :57 (c2 = at·c1, with `at` never formed),
// :90 (Q1^T·A·Q2), :94 (U = Q1·Q). tcgen05 has no f64 kind, so FP64 tensor work on B200 is
// DMMA; the probe in tools/fp64_peak.cu measured DMMA and DFMA both at ~36.5-37 TFLOP/s.
//
// Tiling: CTA tile BM x BN (warp tile 32x32 = 2x4 DMMA tiles), BK = 32 K-slab, STAGES-deep
// cp.async ring in padded shared memory (row strides chosen so every fragment load is
// 2 wavefronts, the minimum for 256 B). A is streamed once from HBM; X (n x d) comes from L2.
// Small-M shapes split K over gridDim.z with a fixed-order second-stage reduce.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int kBK = 32;
constexpr int kStages = 3;

template <int BM, int BN, bool TRANS>
struct Smem {
    // op N: A tile stored [BM][BK+4]  (stride = 4 mod 16 doubles -> conflict-free (g,t) reads)
    // op T: A tile stored [BK][BM+8]  (stride = 8 mod 16 doubles)
    static constexpr int a_stride = TRANS ? BM + 8 : kBK + 4;
    static constexpr int a_elems = TRANS ? kBK * a_stride : BM * a_stride;
    static constexpr int x_stride = BN + 8;
    static constexpr int x_elems = kBK * x_stride;
    static constexpr int stage_elems = a_elems + x_elems;
    static constexpr int bytes = kStages * stage_elems * 8;
};

template <int BM, int BN, bool TRANS, int VEC>
__device__ __forceinline__ void load_stage(double* sa, double* sx, const double* __restrict__ A, int64_t lda,
                                           const double* __restrict__ X, int64_t ldx, int64_t m0, int64_t k0,
                                           int64_t n0, int64_t Mo, int64_t K, int N, int tid) {
    using S = Smem<BM, BN, TRANS>;
    constexpr int NT = (BM / 32) * (BN / 32) * 32;
    // ---- A tile
    if constexpr (!TRANS) {
        constexpr int CPR = kBK / VEC;  // chunks per row
        for (int c = tid; c < BM * CPR; c += NT) {
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
        constexpr int CPR = BM / VEC;
        for (int c = tid; c < kBK * CPR; c += NT) {
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
    // ---- X tile [BK][BN] (X rows are 16-B aligned: ldx is even by construction)
    {
        constexpr int CPR = BN / 2;
        for (int c = tid; c < kBK * CPR; c += NT) {
            const int r = c / CPR, cc = (c % CPR) * 2;
            const int64_t gr = k0 + r, gc = n0 + cc;
            int bytes = 0;
            const double* src = X;
            if (gr < K && gc < N) {
                bytes = int(imin64(2, N - gc)) * 8;
                src = X + gr * ldx + gc;
            }
            cp_async_zfill<16>(sx + r * S::x_stride + cc, src, bytes);
        }
    }
}

template <int BM, int BN, bool TRANS, int VEC>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32)
    k_gemm_f64(const double* __restrict__ A, int64_t lda, const double* __restrict__ X, int64_t ldx,
               double* __restrict__ C, int64_t ldc, int64_t split_stride, int64_t Mo, int64_t K, int N,
               int ktiles_per_split) {
    using S = Smem<BM, BN, TRANS>;
    constexpr int WN = BN / 32;
    constexpr int NT = (BM / 32) * WN * 32;
    extern __shared__ __align__(16) double smem[];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / WN) * 32, wn0 = (warp % WN) * 32;
    const int64_t m0 = int64_t(blockIdx.x) * BM;
    const int64_t n0 = int64_t(blockIdx.y) * BN;
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int64_t kt_begin = int64_t(blockIdx.z) * ktiles_per_split;
    const int64_t kt_end = imin64(ktiles, kt_begin + ktiles_per_split);
    const int nk = int(imax64(0, kt_end - kt_begin));
    C += int64_t(blockIdx.z) * split_stride;

    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) {
            double* sa = smem + s * S::stage_elems;
            load_stage<BM, BN, TRANS, VEC>(sa, sa + S::a_elems, A, lda, X, ldx, m0, (kt_begin + s) * kBK, n0,
                                           Mo, K, N, tid);
        }
        cp_async_commit();
    }

    for (int it = 0; it < nk; ++it) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int nxt = it + kStages - 1;
            if (nxt < nk) {
                double* sa = smem + (nxt % kStages) * S::stage_elems;
                load_stage<BM, BN, TRANS, VEC>(sa, sa + S::a_elems, A, lda, X, ldx, m0, (kt_begin + nxt) * kBK,
                                               n0, Mo, K, N, tid);
            }
            cp_async_commit();
        }
        const double* sa = smem + (it % kStages) * S::stage_elems;
        const double* sx = sa + S::a_elems;
#pragma unroll
        for (int kk = 0; kk < kBK; kk += 8) {
            double af[2][4], bf[4][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = wm0 + mt * 16 + g;
                if constexpr (!TRANS) {
                    af[mt][0] = sa[r * S::a_stride + kk + t];
                    af[mt][1] = sa[(r + 8) * S::a_stride + kk + t];
                    af[mt][2] = sa[r * S::a_stride + kk + t + 4];
                    af[mt][3] = sa[(r + 8) * S::a_stride + kk + t + 4];
                } else {
                    af[mt][0] = sa[(kk + t) * S::a_stride + r];
                    af[mt][1] = sa[(kk + t) * S::a_stride + r + 8];
                    af[mt][2] = sa[(kk + t + 4) * S::a_stride + r];
                    af[mt][3] = sa[(kk + t + 4) * S::a_stride + r + 8];
                }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int c = wn0 + nt * 8 + g;
                bf[nt][0] = sx[(kk + t) * S::x_stride + c];
                bf[nt][1] = sx[(kk + t + 4) * S::x_stride + c];
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma_16x8x8(acc[mt][nt], af[mt], bf[nt]);
        }
    }
    cp_async_wait<0>();

    // Epilogue: rows (g, g+8), cols (2t, 2t+1) of each 16x8 tile.
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t row = m0 + wm0 + mt * 16 + g + h * 8;
            if (row >= Mo) continue;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int64_t col = n0 + wn0 + nt * 8 + 2 * t;
                double* dst = C + row * ldc + col;
                if (col + 1 < N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                    *reinterpret_cast<double2*>(dst) = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
                } else if (col < N) {
                    dst[0] = acc[mt][nt][2 * h];
                    if (col + 1 < N) dst[1] = acc[mt][nt][2 * h + 1];
                }
            }
        }
    }
}

// C = sum_{s < splits} P[s] in increasing s (fixed order => replicas are bit-identical).
// Partials are packed Mo x N; C has leading dimension ldc.
__global__ void k_reduce_splits_f64(const double* __restrict__ P, int64_t split_stride, int splits,
                                    double* __restrict__ C, int64_t ldc, int64_t rows, int N) {
    const int64_t total = rows * N;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        double s = P[e];
        for (int k = 1; k < splits; ++k) s += P[k * split_stride + e];
        C[(e / N) * ldc + e % N] = s;
    }
}

template <int BM, int BN, bool TRANS>
cudaError_t launch(const double* A, int64_t lda, const double* X, int64_t ldx, double* C, int64_t ldc,
                   int64_t split_stride, int64_t Mo, int64_t K, int N, int splits, int kps, cudaStream_t st) {
    using S = Smem<BM, BN, TRANS>;
    const int NT = (BM / 32) * (BN / 32) * 32;
    dim3 grid(unsigned((Mo + BM - 1) / BM), unsigned((N + BN - 1) / BN), unsigned(splits));
    const bool vec = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
    if (vec) {
        auto k = k_gemm_f64<BM, BN, TRANS, 2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::bytes);
        k<<<grid, NT, S::bytes, st>>>(A, lda, X, ldx, C, ldc, split_stride, Mo, K, N, kps);
    } else {
        auto k = k_gemm_f64<BM, BN, TRANS, 1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::bytes);
        k<<<grid, NT, S::bytes, st>>>(A, lda, X, ldx, C, ldc, split_stride, Mo, K, N, kps);
    }
    return cudaGetLastError();
}

void tile_shape(Op op, int N, int& bm, int& bn) {
    if (N <= 32) { bn = 32; bm = 128; }
    else if (N <= 64) { bn = 64; bm = 64; }
    else { bn = 128; bm = 64; }
    (void)op;
}

}  // namespace

GemmPlan plan_gemm_f64(Op op, int64_t Mo, int64_t K, int N, int num_sms) {
    GemmPlan p;
    tile_shape(op, N, p.bm, p.bn);
    const int64_t tiles = ((Mo + p.bm - 1) / p.bm) * ((N + p.bn - 1) / p.bn);
    const int64_t ktiles = (K + kBK - 1) / kBK;
    // Per-SM work model: an SM's FP64 pipe is shared by its resident CTAs, so the makespan is
    // ceil(CTAs / SMs) CTA-works of size 1/splits. Small penalty per split for partial traffic.
    double best = 1e30;
    int best_s = 1;
    const int max_s = int(imax64(1, imin64(ktiles / 4, 32)));
    for (int s = 1; s <= max_s; ++s) {
        const double waves = std::ceil(double(tiles) * s / num_sms);
        const double cost = waves / s * (1.0 + 0.01 * (s - 1)) + (s > 1 ? 0.02 : 0.0);
        if (cost < best - 1e-12) { best = cost; best_s = s; }
    }
    p.splits = best_s;
    const int64_t kps = (ktiles + p.splits - 1) / p.splits;
    p.splits = int((ktiles + kps - 1) / kps);  // no empty splits
    p.ws_elems = p.splits > 1 ? int64_t(p.splits) * Mo * N : 0;
    return p;
}

cudaError_t gemm_f64(Op op, const double* A, int64_t lda, const double* X, int64_t ldx, double* C, int64_t ldc,
                     int64_t Mo, int64_t K, int N, const GemmPlan& p, double* ws, cudaStream_t st) {
    if (Mo <= 0 || N <= 0) return cudaSuccess;
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int kps = int((ktiles + p.splits - 1) / p.splits);
    double* out = p.splits > 1 ? ws : C;
    const int64_t ldo = p.splits > 1 ? N : ldc;
    const int64_t sstride = Mo * N;
    cudaError_t e;
#define CORU_GEMM_CASE(BM_, BN_)                                                                          \
    if (p.bm == BM_ && p.bn == BN_) {                                                                     \
        e = op == Op::N ? launch<BM_, BN_, false>(A, lda, X, ldx, out, ldo, sstride, Mo, K, N, p.splits, kps, st) \
                        : launch<BM_, BN_, true>(A, lda, X, ldx, out, ldo, sstride, Mo, K, N, p.splits, kps, st);  \
    } else
    CORU_GEMM_CASE(128, 32) CORU_GEMM_CASE(64, 64) CORU_GEMM_CASE(64, 128) { return cudaErrorInvalidValue; }
#undef CORU_GEMM_CASE
    if (e != cudaSuccess) return e;
    if (p.splits > 1) {
        // partials are packed Mo x N; reduce into C (ldc)
        const int64_t total = Mo * N;
        const int threads = 256;
        const int blocks = int(imin64((total + threads - 1) / threads, 148 * 8));
        k_reduce_splits_f64<<<blocks, threads, 0, st>>>(ws, sstride, p.splits, C, ldc, Mo, N);
        e = cudaGetLastError();
    }
    return e;
}

}  // namespace coru_gpu
