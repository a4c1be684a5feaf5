// Wide-sketch QR (d > 128: BASELINE C4 d = 220 fp64, C5 d = 520 fp32) by CholeskyQR2 in fp64,
// with an automatic fall-back to the Householder TSQR tree.
//
// householder_qr (qr.hpp:85-99) at corutv.hpp:59-60 computes the unique QR of the sketch with a
// positive diagonal; any backward-stable QR of a full-rank input returns the same Q and R up to
// rounding. For wide sketches the Householder tree is d sequential reflector steps per level on a
// single SM (C5: ~0.5 s per decomposition), while CholeskyQR2 is three GEMM-shaped passes:
//   G = X^T X (FP64 DMMA, reduction over all m rows)  ->  G = L L^T (blocked Cholesky, one CTA,
//   DMMA trailing updates)  ->  Q = X R^{-1}, R = L^T (row-block triangular solve, DMMA),
// applied twice (the second pass restores orthogonality to fp64 level), R = R2·R1.
// In fp64 arithmetic this is accurate for cond(X) up to ~1e7 (Yamamoto et al., CholeskyQR2);
// the fp32 sketch is widened to fp64 first. The kernels write a status word: a non-positive
// Cholesky pivot, an estimated cond(X) = max r_ii / min r_ii above 1e6 in the first pass, or a
// second-pass diagonal away from 1 sets it, and the gated Householder kernels then recompute Q and
// R on the device (no host synchronisation): the result is always the Householder-quality QR.
#include <algorithm>
#include <cmath>

#include "cholqr.cuh"
#include "common.cuh"
#include "cta_blas.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

constexpr int kCholThreads = 512;
constexpr int kCholNB = 32;
constexpr int kTrsmRows = 32;
constexpr int kTrsmThreads = 256;
constexpr int kCholScratch = 4096;

template <typename T>
__global__ void k_widen(const T* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd, int64_t rows,
                        int cols) {
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols;
        const int c = int(e % cols);
        dst[r * ldd + c] = double(src[r * lds + c]);
    }
}

// Trailing update of the blocked Cholesky: C(i,j) -= sum_k L(i,k) L(j,k) for the 16 x 8 tiles that
// touch the lower triangle (the only part later panels read), C (nt x nt, row-major, ldc) in GLOBAL
// memory, L (nt x K, K <= 32, row-major, ldl) in shared memory. A warp owns 16-row strips: the
// strip's L fragments are loaded once and reused by its tiles, which are processed four at a time
// with their C entries requested before the DMMAs. The generic cta_mm_f64 updated all nt^2 entries
// one tile at a time behind a dependent L2 read-modify-write each (2.3 ms per 520 x 520 factor).
// Same k order and the same c + (-1)·acc per entry: bit-identical on the lower triangle.
__device__ __forceinline__ void cta_syrk_lower_global(int nt, int K, const double* L, int ldl, double* __restrict__ C,
                                                      int ldc) {
    const int lane = threadIdx.x & 31, warp = int(threadIdx.x >> 5), nw = int(blockDim.x >> 5);
    const int g = lane >> 2, t = lane & 3;
    const int tm = (nt + 15) >> 4, tn = (nt + 7) >> 3;
    constexpr int TB = 4;
    for (int ti = warp; ti < tm; ti += nw) {
        const int ia = (ti << 4) + g, ib = ia + 8;
        double a[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k0 = 8 * u + t, k1 = k0 + 4;
            a[u][0] = (ia < nt && k0 < K) ? L[ia * ldl + k0] : 0.0;
            a[u][1] = (ib < nt && k0 < K) ? L[ib * ldl + k0] : 0.0;
            a[u][2] = (ia < nt && k1 < K) ? L[ia * ldl + k1] : 0.0;
            a[u][3] = (ib < nt && k1 < K) ? L[ib * ldl + k1] : 0.0;
        }
        const int ntj = min(tn, 2 * ti + 2);  // tiles with a column <= the strip's last row
        for (int tj0 = 0; tj0 < ntj; tj0 += TB) {
            double cold[TB][4], acc[TB][4];
#pragma unroll
            for (int b = 0; b < TB; ++b)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = (ti << 4) + g + ((e >> 1) << 3), j = ((tj0 + b) << 3) + 2 * t + (e & 1);
                    acc[b][e] = 0.0;
                    cold[b][e] = (tj0 + b < ntj && i < nt && j < nt) ? C[int64_t(i) * ldc + j] : 0.0;
                }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (8 * u >= K) break;
                const int k0 = 8 * u + t, k1 = k0 + 4;
#pragma unroll
                for (int b = 0; b < TB; ++b) {
                    const int jb = ((tj0 + b) << 3) + g;
                    double bb[2];
                    bb[0] = (tj0 + b < ntj && jb < nt && k0 < K) ? L[jb * ldl + k0] : 0.0;
                    bb[1] = (tj0 + b < ntj && jb < nt && k1 < K) ? L[jb * ldl + k1] : 0.0;
                    dmma_16x8x8(acc[b], a[u], bb);
                }
            }
#pragma unroll
            for (int b = 0; b < TB; ++b)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = (ti << 4) + g + ((e >> 1) << 3), j = ((tj0 + b) << 3) + 2 * t + (e & 1);
                    if (tj0 + b < ntj && i < nt && j < nt) C[int64_t(i) * ldc + j] = cold[b][e] + (-1.0) * acc[b][e];
                }
        }
    }
}

// Blocked right-looking Cholesky of the d x d Gram matrix (row-major, ld ldg, overwritten), one CTA.
// Outputs R = L^T (row-major, upper, exact zeros below) and, per 32-column block, the inverse of
// the diagonal block of R (RinvD[blk], 32 x 32 row-major upper). status |= 1 on a non-positive
// or non-finite pivot, |= 2 (pass 0) when max r_ii / min r_ii > 1e6, |= 4 (pass 1) when some
// r_ii is outside [0.5, 2] (the first pass did not orthonormalise).
__global__ void __launch_bounds__(kCholThreads, 1)
    k_chol_blocked(double* __restrict__ G, int ldg, int d, double* __restrict__ R, int ldr,
                   double* __restrict__ RinvD, int* __restrict__ status, int pass) {
    extern __shared__ __align__(16) double csm[];
    constexpr int NB = kCholNB, LDL = NB + 1;
    const int ldp = NB + 1;
    double* P = csm;                          // panel, nr x NB (ld ldp)
    double* Li = P + size_t(d) * ldp;         // inverse of the diagonal block, NB x LDL (lower)
    __shared__ int bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) bad = 0;
    for (int e = tid; e < d * d; e += kCholThreads) {
        const int r = e / d, c = e % d;
        if (r > c) R[int64_t(r) * ldr + c] = 0.0;
    }
    __syncthreads();
    for (int p0 = 0; p0 < d; p0 += NB) {
        const int nb = min(NB, d - p0), nr = d - p0;
        for (int e = tid; e < nr * nb; e += kCholThreads) {
            const int r = e / nb, c = e % nb;
            P[r * ldp + c] = G[int64_t(p0 + r) * ldg + p0 + c];
        }
        __syncthreads();
        if (warp == 0) {
            // unblocked Cholesky of the nb x nb diagonal block: lane r owns row r
            for (int j = 0; j < nb; ++j) {
                const double piv = P[j * ldp + j];
                if (!(piv > 0.0) || !isfinite(piv)) {
                    if (lane == 0) bad = 1;
                    break;
                }
                const double ljj = sqrt(piv);
                __syncwarp();
                if (lane == j) P[j * ldp + j] = ljj;
                if (lane > j && lane < nb) P[lane * ldp + j] /= ljj;
                __syncwarp();
                if (lane > j && lane < nb) {
                    const double lrj = P[lane * ldp + j];
                    for (int k = j + 1; k <= lane; ++k) P[lane * ldp + k] -= lrj * P[k * ldp + j];
                }
                __syncwarp();
            }
            __syncwarp();
            // inverse of the lower diagonal block: lane c forms column c by forward substitution
            if (!bad && lane < nb) {
                const int c = lane;
                for (int i = 0; i < nb; ++i) {
                    double s = (i == c) ? 1.0 : 0.0;
                    for (int k = c; k < i; ++k) s -= P[i * ldp + k] * Li[k * LDL + c];
                    Li[i * LDL + c] = i < c ? 0.0 : s / P[i * ldp + i];
                }
            }
        }
        __syncthreads();
        if (bad) break;
        // panel below the diagonal block: L_ip = G_ip · L_pp^{-T}   (row r: y_c = sum_{k<=c} x_k Li[c][k])
        for (int r = nb + tid; r < nr; r += kCholThreads) {
            double x[NB], y[NB];
#pragma unroll
            for (int k = 0; k < NB; ++k) x[k] = k < nb ? P[r * ldp + k] : 0.0;
#pragma unroll
            for (int c = 0; c < NB; ++c) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k <= c; ++k) s += x[k] * Li[c * LDL + k];
                y[c] = s;
            }
#pragma unroll
            for (int c = 0; c < NB; ++c)
                if (c < nb) P[r * ldp + c] = y[c];
        }
        __syncthreads();
        // R rows [p0, p0+nb): R[p0+c][p0+r] = L[p0+r][p0+c] (r >= c); RinvD block = Li^T
        for (int e = tid; e < nr * nb; e += kCholThreads) {
            const int r = e / nb, c = e % nb;
            if (r >= c) R[int64_t(p0 + c) * ldr + p0 + r] = P[r * ldp + c];
        }
        double* Rb = RinvD + size_t(p0 / NB) * NB * NB;
        for (int e = tid; e < NB * NB; e += kCholThreads) {
            const int i = e / NB, j = e % NB;  // Rinv(i, j) = Li(j, i)
            Rb[e] = (i < nb && j < nb && j >= i) ? Li[j * LDL + i] : 0.0;
        }
        // trailing update G_tt -= L_tp L_tp^T (DMMA)
        const int nt = nr - nb;
        if (nt > 0) cta_syrk_lower_global(nt, nb, P + nb * ldp, ldp, G + int64_t(p0 + nb) * ldg + p0 + nb, ldg);
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0) {
        int st = bad ? 1 : 0;
        if (!bad) {
            double mn = 1e308, mx = 0.0;
            for (int i = 0; i < d; ++i) {
                const double v = R[int64_t(i) * ldr + i];
                mn = fmin(mn, v);
                mx = fmax(mx, v);
            }
            if (pass == 0 && !(mx <= 1e6 * mn)) st |= 2;
            if (pass == 1 && !(mn >= 0.5 && mx <= 2.0)) st |= 4;
        }
        if (pass == 0) *status = st;
        else *status |= st;
    }
}

// Q = X · R^{-1} for 32-row blocks of X (fp64, ld ldx): blocked forward substitution over 32-column
// panels, X_p <- (X_p - X_{<p} R_{<p,p}) · Rinv_pp with DMMA for the off-diagonal part.
template <typename TO>
__global__ void __launch_bounds__(kTrsmThreads, 1)
    k_trsm_rinv(const double* __restrict__ X, int64_t ldx, int64_t m, int d, const double* __restrict__ R, int ldr,
                const double* __restrict__ RinvD, TO* __restrict__ Q, int64_t ldq, double* __restrict__ Q64,
                int64_t ldq64) {
    extern __shared__ __align__(16) double tsm[];
    const int lds = d + 1;
    double* Xs = tsm;                               // kTrsmRows x lds
    double* Ys = Xs + kTrsmRows * lds;              // kTrsmRows x 33 (block result)
    double* scr = Ys + kTrsmRows * 33;
    const int tid = threadIdx.x;
    const int64_t r0 = int64_t(blockIdx.x) * kTrsmRows;
    const int rows = int(m - r0 < kTrsmRows ? m - r0 : kTrsmRows);
    for (int e = tid; e < kTrsmRows * d; e += kTrsmThreads) {
        const int r = e / d, c = e % d;
        // X == nullptr: rows of the identity (the result is then R^{-1} itself)
        Xs[r * lds + c] = r < rows ? (X ? X[(r0 + r) * ldx + c] : (r0 + r == c ? 1.0 : 0.0)) : 0.0;
    }
    __syncthreads();
    for (int p0 = 0; p0 < d; p0 += kCholNB) {
        const int nb = min(kCholNB, d - p0);
        if (p0 > 0) {
            cta_mm_f64(kTrsmRows, nb, p0, Xs, lds, 1, R + p0, ldr, 1, Xs + p0, lds, 1, -1.0, true, scr, 2048);
            __syncthreads();
        }
        const double* Rb = RinvD + size_t(p0 / kCholNB) * kCholNB * kCholNB;
        for (int e = tid; e < kTrsmRows * kCholNB; e += kTrsmThreads) {
            const int r = e / kCholNB, c = e % kCholNB;
            double s = 0.0;
            if (c < nb)
                for (int k = 0; k <= c; ++k) s += Xs[r * lds + p0 + k] * Rb[k * kCholNB + c];
            Ys[r * 33 + c] = s;
        }
        __syncthreads();
        for (int e = tid; e < kTrsmRows * nb; e += kTrsmThreads) {
            const int r = e / nb, c = e % nb;
            Xs[r * lds + p0 + c] = Ys[r * 33 + c];
        }
        __syncthreads();
    }
    for (int e = tid; e < rows * d; e += kTrsmThreads) {
        const int r = e / d, c = e % d;
        const double v = Xs[r * lds + c];
        Q[(r0 + r) * ldq + c] = TO(v);
        if (Q64) Q64[(r0 + r) * ldq64 + c] = v;
    }
}

template <typename T>
__global__ void k_narrow_square(const double* __restrict__ src, int lds, int d, T* __restrict__ dst, int ldd) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d * d; e += gridDim.x * blockDim.x)
        dst[(e / d) * ldd + e % d] = T(src[(e / d) * lds + e % d]);
}

template <typename T>
__global__ void k_narrow_rect(const double* __restrict__ src, int64_t lds, int64_t rows, int cols, T* __restrict__ dst,
                              int64_t ldd) {
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols;
        const int c = int(e % cols);
        dst[r * ldd + c] = T(src[r * lds + c]);
    }
}

size_t chol_smem(int d) { return (size_t(d) * (kCholNB + 1) + kCholNB * (kCholNB + 1) + kCholScratch) * 8; }
size_t trsm_smem(int d) { return (size_t(kTrsmRows) * (d + 1) + kTrsmRows * 33 + 2048) * 8; }

}  // namespace

bool cholqr_applicable(int64_t m, int d, int max_smem) {
    return d > 128 && d <= 1024 && m >= 2 * int64_t(d) && chol_smem(d) <= size_t(max_smem) &&
           trsm_smem(d) <= size_t(max_smem);
}

CholQrPlan plan_cholqr(int64_t m, int d, size_t eb, int num_sms) {
    CholQrPlan p;
    p.m = m;
    p.d = d;
    p.ldw = d + (d & 1);
    p.xd_elems = eb == 8 ? 0 : m * p.ldw;  // fp64 copy of an fp32 sketch
    p.q1_elems = m * p.ldw;
    p.gram_ws = std::max({plan_gemm_f64(Op::T, d, m, d, num_sms).ws_elems, plan_gemm_f64(Op::N, d, d, d, num_sms).ws_elems,
                          plan_gemm_f64(Op::N, m, d, d, num_sms).ws_elems});
    p.dd_elems = int64_t(d) * p.ldw;  // d x d fp64 matrices with an even row stride (16-byte rows)
    p.rinvd_elems = int64_t((d + kCholNB - 1) / kCholNB) * kCholNB * kCholNB;
    return p;
}

int64_t cholqr_ws_doubles(const CholQrPlan& p) {
    return p.xd_elems + p.q1_elems + p.gram_ws + 4 * p.dd_elems + 2 * p.rinvd_elems + 1;
}

template <typename T>
cudaError_t cholqr_factor(const CholQrPlan& p, const T* B, int64_t ldb, double* ws, int* status, T* r_out, int max_smem,
                          int num_sms, cudaStream_t st, const CholQrReduce* reduce) {
    const int64_t m = p.m;
    const int d = p.d;
    double* xd = ws;
    double* q1 = xd + p.xd_elems;
    double* gws = q1 + p.q1_elems;
    double* G = gws + p.gram_ws;
    double* R1 = G + p.dd_elems;
    double* R2 = R1 + p.dd_elems;
    double* Rf = R2 + p.dd_elems;
    double* RinvD1 = Rf + p.dd_elems;
    double* RinvD2 = RinvD1 + p.rinvd_elems;
    const double* X;
    int64_t ldx;
    if constexpr (sizeof(T) == 8) {
        X = reinterpret_cast<const double*>(B);
        ldx = ldb;
    } else {
        const int blocks = int(std::min<int64_t>((m * d + 255) / 256, int64_t(num_sms) * 16));
        k_widen<T><<<blocks, 256, 0, st>>>(B, ldb, xd, p.ldw, m, d);
        X = xd;
        ldx = p.ldw;
    }
    allow_max_smem(k_chol_blocked);
    allow_max_smem(k_trsm_rinv<double>);
    cudaError_t e;
    // pass 1: G = X^T X, R1, Q1 = X R1^{-1} (fp64)
    GemmPlan gp = plan_gemm_f64(Op::T, d, m, d, num_sms);
    const int ldw = p.ldw;
    if ((e = gemm_f64(Op::T, X, ldx, X, ldx, G, ldw, d, m, d, gp, gws, st)) != cudaSuccess) return e;
    if (reduce && (e = (*reduce)(G, size_t(d) * size_t(ldw))) != cudaSuccess) return e;
    k_chol_blocked<<<1, kCholThreads, chol_smem(d), st>>>(G, ldw, d, R1, ldw, RinvD1, status, 0);
    // Q1 = X R1^{-1} as a GEMM with the explicit inverse: R1^{-1} = I · R1^{-1} by the blocked
    // substitution kernel on the d rows of the identity (G is free between the two Gram products
    // and holds it), then one stream-K DMMA product. The substitution kernel over all m rows ran at
    // 6 TFLOP/s (C5, 65536 x 520: 2.8 ms per solve against 1.4 ms this way).
    const unsigned tbi = unsigned((d + kTrsmRows - 1) / kTrsmRows);
    const GemmPlan qp = plan_gemm_f64(Op::N, m, d, d, num_sms);
    k_trsm_rinv<double><<<tbi, kTrsmThreads, trsm_smem(d), st>>>(nullptr, 0, d, d, R1, ldw, RinvD1, G, ldw, nullptr, 0);
    if ((e = gemm_f64(Op::N, X, ldx, G, ldw, q1, ldw, m, d, d, qp, gws, st)) != cudaSuccess) return e;
    // pass 2: G = Q1^T Q1, R2; R = R2 R1 (Q = Q1 R2^{-1} is formed by cholqr_form_q)
    if ((e = gemm_f64(Op::T, q1, ldw, q1, ldw, G, ldw, d, m, d, gp, gws, st)) != cudaSuccess) return e;
    if (reduce && (e = (*reduce)(G, size_t(d) * size_t(ldw))) != cudaSuccess) return e;
    k_chol_blocked<<<1, kCholThreads, chol_smem(d), st>>>(G, ldw, d, R2, ldw, RinvD2, status, 1);
    // R2^{-1} for cholqr_form_q, again in G (dead from here on)
    k_trsm_rinv<double><<<tbi, kTrsmThreads, trsm_smem(d), st>>>(nullptr, 0, d, d, R2, ldw, RinvD2, G, ldw, nullptr, 0);
    GemmPlan rp = plan_gemm_f64(Op::N, d, d, d, num_sms);
    if ((e = gemm_f64(Op::N, R2, ldw, R1, ldw, Rf, ldw, d, d, d, rp, gws, st)) != cudaSuccess) return e;
    k_narrow_square<T><<<std::max(1, std::min(num_sms * 4, (d * d + 255) / 256)), 256, 0, st>>>(Rf, ldw, d, r_out, d);
    (void)max_smem;
    return cudaGetLastError();
}

template <typename T>
cudaError_t cholqr_form_q(const CholQrPlan& p, double* ws, T* Q, int64_t ldq, int num_sms, cudaStream_t st) {
    const int64_t m = p.m;
    const int d = p.d;
    double* xd = ws;
    double* q1 = ws + p.xd_elems;
    double* gws = q1 + p.q1_elems;
    double* G = gws + p.gram_ws;  // R2^{-1} (cholqr_factor)
    const GemmPlan qp = plan_gemm_f64(Op::N, m, d, d, num_sms);
    if constexpr (sizeof(T) == 8) {
        return gemm_f64(Op::N, q1, p.ldw, G, p.ldw, reinterpret_cast<double*>(Q), ldq, m, d, d, qp, gws, st);
    } else {
        // fp32 sketch: the product in fp64 into the (now free) widened copy of the sketch, then narrowed
        cudaError_t e = gemm_f64(Op::N, q1, p.ldw, G, p.ldw, xd, p.ldw, m, d, d, qp, gws, st);
        if (e != cudaSuccess) return e;
        const int blocks = int(std::min<int64_t>((m * d + 255) / 256, int64_t(num_sms) * 16));
        k_narrow_rect<T><<<blocks, 256, 0, st>>>(xd, p.ldw, m, d, Q, ldq);
        return cudaGetLastError();
    }
}

int cholqr_launches(int d) {
    (void)d;
    return 11;
}

#define CORU_INST(T)                                                                                               \
    template cudaError_t cholqr_factor<T>(const CholQrPlan&, const T*, int64_t, double*, int*, T*, int, int,       \
                                          cudaStream_t, const CholQrReduce*);                                     \
    template cudaError_t cholqr_form_q<T>(const CholQrPlan&, double*, T*, int64_t, int, cudaStream_t);
CORU_INST(double)
CORU_INST(float)
#undef CORU_INST

}  // namespace coru_gpu
