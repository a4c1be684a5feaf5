// FP32 skinny GEMM (CUDA-core FFMA) for the fp32 configuration (BASELINE config 5).
//
// Same contract as gemm_f64 (op N: C = A·X, op T: C = A^T·X without forming A^T; deterministic
// fixed-order split-K). Exact fp32 arithmetic: the north_star's fp32 tolerance (1e-4 relative
// error / 1e-3 |diag T|) is specified against an fp32 run of the reference algorithm, which
// single-pass TF32 tensor cores (10-bit mantissa) cannot meet (SURVEY.md §7 hard part 6).
//
// Tiling: CTA tile 128 x 64, 256 threads, 8 x 4 register tile per thread, BK = 16 slabs staged
// k-major in shared memory (A transposed on the way in for op N) through a 3-deep cp.async ring.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

constexpr int kBM = 128, kBN = 64, kBK = 16, kTM = 8, kTN = 4, kThreads = 256, kStages = 3;
constexpr int kAS = kBM + 4;  // k-major A tile row stride (floats)
constexpr int kXS = kBN + 4;
constexpr int kStageFloats = kBK * kAS + kBK * kXS;

__host__ __device__ inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

template <bool TRANS>
__device__ __forceinline__ void load_stage_f32(float* sa, float* sx, const float* __restrict__ A, int64_t lda,
                                               const float* __restrict__ X, int64_t ldx, int64_t m0, int64_t k0,
                                               int64_t n0, int64_t Mo, int64_t K, int N, int tid) {
    if constexpr (!TRANS) {
        // A rows [m0, m0+BM) x cols [k0, k0+BK): read 4-byte elements, store transposed (k-major).
        for (int e = tid; e < kBM * kBK; e += kThreads) {
            const int r = e / kBK, c = e % kBK;
            const int64_t gr = m0 + r, gc = k0 + c;
            const bool ok = gr < Mo && gc < K;
            cp_async_zfill<4>(sa + c * kAS + r, ok ? A + gr * lda + gc : A, ok ? 4 : 0);
        }
    } else {
        // A rows [k0, k0+BK) x cols [m0, m0+BM): already k-major.
        for (int e = tid; e < kBK * kBM; e += kThreads) {
            const int r = e / kBM, c = e % kBM;
            const int64_t gr = k0 + r, gc = m0 + c;
            const bool ok = gr < K && gc < Mo;
            cp_async_zfill<4>(sa + r * kAS + c, ok ? A + gr * lda + gc : A, ok ? 4 : 0);
        }
    }
    for (int e = tid; e < kBK * kBN; e += kThreads) {
        const int r = e / kBN, c = e % kBN;
        const int64_t gr = k0 + r, gc = n0 + c;
        const bool ok = gr < K && gc < N;
        cp_async_zfill<4>(sx + r * kXS + c, ok ? X + gr * ldx + gc : X, ok ? 4 : 0);
    }
}

template <bool TRANS>
__global__ void __launch_bounds__(kThreads) k_gemm_f32(const float* __restrict__ A, int64_t lda,
                                                       const float* __restrict__ X, int64_t ldx, float* __restrict__ C,
                                                       int64_t ldc, int64_t split_stride, int64_t Mo, int64_t K, int N,
                                                       int ktiles_per_split) {
    extern __shared__ __align__(16) float fsm[];
    const int tid = threadIdx.x;
    const int tx = tid % (kBN / kTN), ty = tid / (kBN / kTN);  // 16 x 16 thread grid
    const int64_t m0 = int64_t(blockIdx.x) * kBM, n0 = int64_t(blockIdx.y) * kBN;
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int64_t kt0 = int64_t(blockIdx.z) * ktiles_per_split;
    const int nk = int(imin(ktiles, kt0 + ktiles_per_split) - kt0);
    C += int64_t(blockIdx.z) * split_stride;
    float acc[kTM][kTN];
#pragma unroll
    for (int i = 0; i < kTM; ++i)
#pragma unroll
        for (int j = 0; j < kTN; ++j) acc[i][j] = 0.f;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) {
            float* sa = fsm + s * kStageFloats;
            load_stage_f32<TRANS>(sa, sa + kBK * kAS, A, lda, X, ldx, m0, (kt0 + s) * kBK, n0, Mo, K, N, tid);
        }
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        const int nxt = it + kStages - 1;
        if (nxt < nk) {
            float* sa = fsm + (nxt % kStages) * kStageFloats;
            load_stage_f32<TRANS>(sa, sa + kBK * kAS, A, lda, X, ldx, m0, (kt0 + nxt) * kBK, n0, Mo, K, N, tid);
        }
        cp_async_commit();
        const float* sa = fsm + (it % kStages) * kStageFloats;
        const float* sx = sa + kBK * kAS;
#pragma unroll
        for (int k = 0; k < kBK; ++k) {
            float a[kTM], b[kTN];
            const float4 a0 = *reinterpret_cast<const float4*>(sa + k * kAS + ty * 4);
            const float4 a1 = *reinterpret_cast<const float4*>(sa + k * kAS + 64 + ty * 4);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            const float4 b0 = *reinterpret_cast<const float4*>(sx + k * kXS + tx * 4);
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
#pragma unroll
            for (int i = 0; i < kTM; ++i)
#pragma unroll
                for (int j = 0; j < kTN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
        const int64_t row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (row >= Mo) continue;
#pragma unroll
        for (int j = 0; j < kTN; ++j) {
            const int64_t col = n0 + tx * 4 + j;
            if (col < N) C[row * ldc + col] = acc[i][j];
        }
    }
}

__global__ void k_reduce_splits_f32(const float* __restrict__ P, int64_t split_stride, int splits, float* __restrict__ C,
                                    int64_t ldc, int64_t rows, int N) {
    const int64_t total = rows * N;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        float s = P[e];
        for (int k = 1; k < splits; ++k) s += P[k * split_stride + e];
        C[(e / N) * ldc + e % N] = s;
    }
}

}  // namespace

GemmPlan plan_gemm_f32(Op op, int64_t Mo, int64_t K, int N, int num_sms) {
    (void)op;
    GemmPlan p;
    p.bm = kBM;
    p.bn = kBN;
    const int64_t tiles = ((Mo + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
    const int64_t ktiles = (K + kBK - 1) / kBK;
    double best = 1e30;
    int best_s = 1;
    const int max_s = int(std::max<int64_t>(1, std::min<int64_t>(ktiles / 8, 32)));
    for (int s = 1; s <= max_s; ++s) {
        const double waves = std::ceil(double(tiles) * s / (2.0 * num_sms));
        const double cost = waves / s * (1.0 + 0.01 * (s - 1)) + (s > 1 ? 0.02 : 0.0);
        if (cost < best - 1e-12) {
            best = cost;
            best_s = s;
        }
    }
    const int64_t kps = (ktiles + best_s - 1) / best_s;
    p.splits = int((ktiles + kps - 1) / kps);
    p.ws_elems = p.splits > 1 ? int64_t(p.splits) * Mo * N : 0;
    return p;
}

cudaError_t gemm_f32(Op op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C, int64_t ldc, int64_t Mo,
                     int64_t K, int N, const GemmPlan& p, float* ws, cudaStream_t st) {
    if (Mo <= 0 || N <= 0) return cudaSuccess;
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int kps = int((ktiles + p.splits - 1) / p.splits);
    float* out = p.splits > 1 ? ws : C;
    const int64_t ldo = p.splits > 1 ? N : ldc;
    const int64_t sstride = Mo * N;
    const dim3 grid(unsigned((Mo + kBM - 1) / kBM), unsigned((N + kBN - 1) / kBN), unsigned(p.splits));
    const size_t smem = size_t(kStages) * kStageFloats * sizeof(float);
    if (op == Op::N) {
        allow_max_smem(k_gemm_f32<false>);
        k_gemm_f32<false><<<grid, kThreads, smem, st>>>(A, lda, X, ldx, out, ldo, sstride, Mo, K, N, kps);
    } else {
        allow_max_smem(k_gemm_f32<true>);
        k_gemm_f32<true><<<grid, kThreads, smem, st>>>(A, lda, X, ldx, out, ldo, sstride, Mo, K, N, kps);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || p.splits == 1) return e;
    const int64_t total = Mo * N;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 8));
    k_reduce_splits_f32<<<blocks, 256, 0, st>>>(ws, sstride, p.splits, C, ldc, Mo, N);
    return cudaGetLastError();
}

}  // namespace coru_gpu
