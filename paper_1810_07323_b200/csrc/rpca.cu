// ALM robust PCA with the CoR-UTV inner step (rpca.hpp:95-169): the lift fused with the ALM
// update, cor_threshold's truncation, and the reductions of the loop. See rpca.cuh.
#include "rpca.cuh"

#include <algorithm>

#include "common.cuh"

namespace coru_gpu {
namespace {

constexpr int kTile = 64;  // L tile (kTile x kTile) per CTA iteration
constexpr int kKc = 32;    // k-chunk of Tp / Vb staged in shared memory
constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) s += red[w];  // fixed order
    __syncthreads();
    return s;
}

// Each CTA walks tiles blockIdx.x, blockIdx.x + gridDim.x, ... (fixed order). The lift L = Tp·V^T of
// a 64 x 64 tile runs on the FP64 tensor cores (DMMA m16n8k8): warp (wm, wn) of the 4 x 2 layout
// owns rows 16·wm.. and columns 32·wn.. (four 16 x 8 accumulators). Tp / V chunks (64 x 32) are
// loaded into registers one chunk (and one tile) ahead of the MMAs and staged in shared memory with
// a 36-double row stride (conflict-free fragment loads). Two CTAs per SM.
constexpr int kLdT = kKc + 4;   // sT / sV row stride (doubles)
constexpr int kLdM = kTile + 2; // sM / sY row stride (doubles; keeps 16-byte cp.async alignment)
template <bool VEC>
__global__ void __launch_bounds__(kThreads, 2) k_rpca_lift_update(const double* __restrict__ Tp, int64_t ldt,
                                                                  const double* __restrict__ Vb, int64_t ldv, int d,
                                                                  int64_t m, int64_t n, const double* __restrict__ M,
                                                                  int64_t ldm, double* __restrict__ Y, int64_t ldy,
                                                                  double* __restrict__ X, int64_t ldx,
                                                                  double* __restrict__ S, int64_t lds,
                                                                  double* __restrict__ L, int64_t ldl, RpcaStep p,
                                                                  int lift_only, double* __restrict__ parts) {
    extern __shared__ __align__(16) double smem[];
    double* sT = smem;                    // kTile x kLdT
    double* sV = sT + kTile * kLdT;       // kTile x kLdT
    double* sMY = sV + kTile * kLdT;      // [M, Y][kTile x kLdM] (16-byte aligned)
    __shared__ double red[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int64_t tiles_n = (n + kTile - 1) / kTile;
    const int64_t tiles = ((m + kTile - 1) / kTile) * tiles_n;
    double part = 0.0;
    constexpr int kPer = kTile * kKc / kThreads;
    double pT[kPer], pV[kPer];
    auto load_chunk = [&](int64_t tt, int k0) {
        const int64_t ti0 = (tt / tiles_n) * kTile, tj0 = (tt % tiles_n) * kTile;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int e = threadIdx.x + q * kThreads;
            const int r = e / kKc, c = e % kKc;
            const bool kc = k0 + c < d;
            pT[q] = (kc && ti0 + r < m) ? __ldg(Tp + (ti0 + r) * ldt + k0 + c) : 0.0;
            pV[q] = (kc && tj0 + r < n) ? __ldg(Vb + (tj0 + r) * ldv + k0 + c) : 0.0;
        }
    };
    // M and Y of a tile are requested with cp.async at the start of the tile, so their DRAM latency
    // hides under the MMAs (one buffer: two CTAs per SM beat one CTA with a double buffer).
    auto prefetch_my = [&](int64_t tt, int buf) {
        const int64_t ti0 = (tt / tiles_n) * kTile, tj0 = (tt % tiles_n) * kTile;
        double* sM = sMY + buf * 2 * kTile * kLdM;
        double* sY = sM + kTile * kLdM;
        if constexpr (VEC) {
            for (int e = threadIdx.x; e < kTile * kTile / 2; e += kThreads) {
                const int r = e / (kTile / 2), c = 2 * (e % (kTile / 2));
                const int64_t gi = ti0 + r, gj = tj0 + c;
                const bool ok = gi < m && gj < n;  // n even when VEC: a pair is all-in or all-out
                const int64_t gi_c = ok ? gi : 0, gj_c = ok ? gj : 0;
                cp_async_zfill<16>(sM + r * kLdM + c, M + gi_c * ldm + gj_c, ok ? 16 : 0);
                cp_async_zfill<16>(sY + r * kLdM + c, Y + gi_c * ldy + gj_c, ok ? 16 : 0);
            }
        } else {
            for (int e = threadIdx.x; e < kTile * kTile; e += kThreads) {
                const int r = e / kTile, c = e % kTile;
                const int64_t gi = ti0 + r, gj = tj0 + c;
                const bool ok = gi < m && gj < n;
                const int64_t gi_c = ok ? gi : 0, gj_c = ok ? gj : 0;
                cp_async_zfill<8>(sM + r * kLdM + c, M + gi_c * ldm + gj_c, ok ? 8 : 0);
                cp_async_zfill<8>(sY + r * kLdM + c, Y + gi_c * ldy + gj_c, ok ? 8 : 0);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t i0 = (t / tiles_n) * kTile, j0 = (t % tiles_n) * kTile;
        const double* sM = sMY;
        const double* sY = sM + kTile * kLdM;
        if (!lift_only) prefetch_my(t, 0);
        double acc[4][4];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[nb][u] = 0.0;
        if (t == int64_t(blockIdx.x)) load_chunk(t, 0);  // later tiles: issued under the previous MMAs
        for (int k0 = 0; k0 < d; k0 += kKc) {
            __syncthreads();  // the previous chunk's MMAs are done with sT / sV
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int e = threadIdx.x + q * kThreads;
                sT[(e / kKc) * kLdT + e % kKc] = pT[q];
                sV[(e / kKc) * kLdT + e % kKc] = pV[q];
            }
            __syncthreads();
            if (k0 + kKc < d) load_chunk(t, k0 + kKc);
            else if (t + gridDim.x < tiles) load_chunk(t + gridDim.x, 0);
            const int ksteps = (min(kKc, d - k0) + 7) / 8;  // zero-padded columns past d add nothing
            for (int ks = 0; ks < ksteps; ++ks) {
                const int kb = ks * 8;
                const double* ta = sT + (wm * 16 + g) * kLdT + kb + t4;
                const double a[4] = {ta[0], ta[8 * kLdT], ta[4], ta[8 * kLdT + 4]};
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) {
                    const double* vb = sV + (wn * 32 + nb * 8 + g) * kLdT + kb + t4;
                    const double b[2] = {vb[0], vb[4]};
                    dmma_16x8x8(acc[nb], a, b);
                }
            }
        }
        if (!lift_only) {
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
        }
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int li = wm * 16 + g + 8 * (u >> 1);
                const int lj = wn * 32 + nb * 8 + 2 * t4 + (u & 1);
                const int64_t gi = i0 + li, gj = j0 + lj;
                if (gi >= m || gj >= n) continue;
                const double l = acc[nb][u];
                if (lift_only) {
                    L[gi * ldl + gj] = l;
                    continue;
                }
                const double mv = sM[li * kLdM + lj];
                const double yv = sY[li * kLdM + lj];
                const double ml = __dsub_rn(mv, l);                        // m - l        (rpca.hpp:143)
                const double w = __dadd_rn(ml, __dmul_rn(yv, p.inv_mu));   // += y·inv_mu  (:144)
                const double mag = __dsub_rn(fabs(w), p.thresh);           // shrink       (:17-26, :145)
                const double s = mag > 0.0 ? (w > 0.0 ? mag : -mag) : 0.0;
                const double r = __dsub_rn(ml, s);                         // resid        (:147-148)
                const double y2 = __dadd_rn(yv, __dmul_rn(p.mu, r));       // y += mu·resid (:149)
                __stcs(S + gi * lds + gj, s);
                __stcs(Y + gi * ldy + gj, y2);
                __stcs(X + gi * ldx + gj, __dadd_rn(__dsub_rn(mv, s), __dmul_rn(y2, p.inv_mu_next)));  // next x
                part = fma(r, r, part);
            }
        }
        if (!lift_only) __syncthreads();  // sM / sY are refilled by the next tile's prefetch
    }
    if (!lift_only) {
        const double s = block_sum(part, red);
        if (threadIdx.x == 0) parts[blockIdx.x] = s;
    }
}

constexpr size_t kUpdSmem = size_t(2 * kTile * kLdT + 2 * kTile * kLdM) * sizeof(double);

__global__ void __launch_bounds__(kThreads) k_sumsq(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                                    double* __restrict__ parts) {
    __shared__ double red[kThreads / 32];
    double s = 0.0;
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x)
        for (int64_t j = threadIdx.x; j < n; j += kThreads) {
            const double v = A[i * lda + j];
            s = fma(v, v, s);
        }
    s = block_sum(s, red);
    if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_sum_parts(const double* __restrict__ parts, int nparts,
                                                        double* __restrict__ out) {
    __shared__ double red[kThreads / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kThreads) s += parts[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[0] = s;
}

__global__ void k_cor_truncate(const double* __restrict__ T, int64_t ldt, int d, double delta, int lower,
                               double* __restrict__ Tr, int64_t ldtr, int* rank_out) {
    __shared__ int s_r;
    if (threadIdx.x == 0) {
        int r = 0;
        for (int j = 0; j < d; ++j) r += fabs(T[int64_t(j) * ldt + j]) > delta;  // corutv.hpp:128-130
        s_r = r;
        if (rank_out) *rank_out = r;
    }
    __syncthreads();
    const int r = s_r;
    for (int64_t e = threadIdx.x; e < int64_t(d) * d; e += blockDim.x) {
        const int i = int(e / d), j = int(e % d);
        const bool keep = lower ? j < r : i < r;
        Tr[int64_t(i) * ldtr + j] = keep ? T[int64_t(i) * ldt + j] : 0.0;
    }
}

__global__ void k_gram_norms(const double* __restrict__ sig, int p, double* __restrict__ out) {
    if (threadIdx.x != 0) return;
    double nuc = 0.0;
    for (int i = 0; i < p; ++i) nuc += sqrt(fmax(sig[i], 0.0));
    out[0] = sqrt(fmax(sig[0], 0.0));
    out[1] = nuc;
}

__global__ void __launch_bounds__(kThreads) k_count_nonzero(const double* __restrict__ A, int64_t lda, int64_t m,
                                                            int64_t n, unsigned long long* out) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x)
        for (int64_t j = threadIdx.x; j < n; j += kThreads) c += A[i * lda + j] != 0.0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);  // integer: order-independent
}

}  // namespace

int rpca_parts(int64_t m, int64_t n, int sms) {
    const int64_t tiles = ((m + kTile - 1) / kTile) * ((n + kTile - 1) / kTile);
    return int(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(sms) * 2)));  // two CTAs per SM
}

cudaError_t rpca_lift_update(const double* Tp, int64_t ldt, const double* Vb, int64_t ldv, int d, int64_t m,
                             int64_t n, const double* M, int64_t ldm, double* Y, int64_t ldy, double* X, int64_t ldx,
                             double* S, int64_t lds, double* L, int64_t ldl, const RpcaStep& p, bool lift_only,
                             double* parts, int nparts, cudaStream_t st) {
    const bool vec = !lift_only && n % 2 == 0 && ldm % 2 == 0 && ldy % 2 == 0 &&
                     (reinterpret_cast<uintptr_t>(M) & 15) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
    auto kern = vec ? k_rpca_lift_update<true> : k_rpca_lift_update<false>;
    allow_max_smem(kern);
    kern<<<nparts, kThreads, kUpdSmem, st>>>(Tp, ldt, Vb, ldv, d, m, n, M, ldm, Y, ldy, X, ldx, S, lds, L, ldl, p,
                                             lift_only ? 1 : 0, parts);
    return cudaGetLastError();
}

cudaError_t cor_truncate(const double* T, int64_t ldt, int d, double delta, int lower, double* Tr, int64_t ldtr,
                         int* rank_out, cudaStream_t st) {
    k_cor_truncate<<<1, 256, 0, st>>>(T, ldt, d, delta, lower, Tr, ldtr, rank_out);
    return cudaGetLastError();
}

cudaError_t sumsq_parts(const double* A, int64_t lda, int64_t m, int64_t n, double* parts, int nparts,
                        cudaStream_t st) {
    k_sumsq<<<nparts, kThreads, 0, st>>>(A, lda, m, n, parts);
    return cudaGetLastError();
}

cudaError_t sum_parts(const double* parts, int nparts, double* out, cudaStream_t st) {
    k_sum_parts<<<1, kThreads, 0, st>>>(parts, nparts, out);
    return cudaGetLastError();
}

cudaError_t gram_norms(const double* sig, int p, double* out, cudaStream_t st) {
    k_gram_norms<<<1, 32, 0, st>>>(sig, p, out);
    return cudaGetLastError();
}

cudaError_t count_nonzero(const double* A, int64_t lda, int64_t m, int64_t n, unsigned long long* out,
                          cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(m, 148 * 8)));
    k_count_nonzero<<<blocks, kThreads, 0, st>>>(A, lda, m, n, out);
    return cudaGetLastError();
}

}  // namespace coru_gpu
