// CTA-level dense kernels on shared-memory operands, used by the blocked Householder kernels
// (TSQR panels, compact-WY updates, QRCP's Q accumulation).
//
// cta_gemm: C(i,j) <op>= sum_k A(i,k)·B(k,j) for i < M, j < N, k < K, with A/B/C given as
// accessor functors (so implicit unit-diagonal / zero-padded reflector storage needs no copy).
// Threads own TM x TN register tiles; when the tiles cannot occupy the CTA the K range is split
// and the partial tiles are reduced through shared memory in a fixed order (deterministic).
#pragma once
#include "common.cuh"

namespace coru_gpu {

template <int TM, int TN, typename T, class FA, class FB, class FC>
__device__ __forceinline__ void cta_gemm(int M, int N, int K, FA A, FB B, FC C, T* scratch, int scratch_elems) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int tm = (M + TM - 1) / TM, tn = (N + TN - 1) / TN, tiles = tm * tn;
    if (tiles == 0 || K <= 0) return;
    // split-K factor: fill the CTA, keep >= 8 k per split, respect the scratch capacity
    int S = 1;
    if (tiles * 2 <= nt) {
        S = min(nt / tiles, max(1, K / 8));
        const int cap = scratch_elems / max(1, tiles * TM * TN);
        S = max(1, min(S, cap));
    }
    const int work = tiles * S;
    for (int w = tid; w < work; w += nt) {
        const int tile = w % tiles, s = w / tiles;
        const int i0 = (tile / tn) * TM, j0 = (tile % tn) * TN;
        const int k0 = int((int64_t(K) * s) / S), k1 = int((int64_t(K) * (s + 1)) / S);
        T acc[TM][TN];
#pragma unroll
        for (int a = 0; a < TM; ++a)
#pragma unroll
            for (int b = 0; b < TN; ++b) acc[a][b] = T(0);
        for (int k = k0; k < k1; ++k) {
            T av[TM], bv[TN];
#pragma unroll
            for (int a = 0; a < TM; ++a) av[a] = (i0 + a < M) ? A(i0 + a, k) : T(0);
#pragma unroll
            for (int b = 0; b < TN; ++b) bv[b] = (j0 + b < N) ? B(k, j0 + b) : T(0);
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) acc[a][b] += av[a] * bv[b];
        }
        if (S == 1) {
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b)
                    if (i0 + a < M && j0 + b < N) C(i0 + a, j0 + b, acc[a][b]);
        } else {
            T* p = scratch + (int64_t(s) * tiles + tile) * (TM * TN);
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) p[a * TN + b] = acc[a][b];
        }
    }
    if (S > 1) {
        __syncthreads();
        for (int e = tid; e < tiles * TM * TN; e += nt) {
            const int tile = e / (TM * TN), r = e % (TM * TN);
            const int i = (tile / tn) * TM + r / TN, j = (tile % tn) * TN + r % TN;
            T v = scratch[e];
            for (int s = 1; s < S; ++s) v += scratch[int64_t(s) * tiles * TM * TN + e];
            if (i < M && j < N) C(i, j, v);
        }
    }
}

// FP64 tensor-core CTA GEMM on shared (or global) operands with explicit element strides:
//   C(i,j) = alpha * sum_k A(i,k) B(k,j) + (accumulate ? C(i,j) : 0)
//   A(i,k) = A[i*ars + k*acs], B(k,j) = B[k*brs + j*bcs], C(i,j) = C[i*crs + j*ccs]
// Warps own 16x8 DMMA tiles (m16n8k8); when the tiles cannot occupy the warps the K range is
// split and the partial tiles are reduced in a fixed order through `scratch` (deterministic).
// Must be called by every thread of the CTA; inputs must be visible (synchronised) on entry and
// outputs are visible to all threads only after the caller's next __syncthreads().
// warp0/nwarps: the participating warps (default: the whole CTA). With a subset, the split-K
// reduction synchronises them through named barrier `bar_id` instead of __syncthreads.
__device__ __forceinline__ void cta_mm_f64(int M, int N, int K, const double* A, int ars, int acs, const double* B,
                                           int brs, int bcs, double* C, int crs, int ccs, double alpha,
                                           bool accumulate, double* scratch, int scratch_elems, int warp0 = 0,
                                           int nwarps = -1, int bar_id = 15) {
    const int lane = threadIdx.x & 31;
    const int all = int(blockDim.x >> 5);
    const int nw = nwarps < 0 ? all : nwarps;
    const int warp = int(threadIdx.x >> 5) - warp0;
    if (warp < 0 || warp >= nw) return;
    const int g = lane >> 2, t = lane & 3;
    const int tm = (M + 15) >> 4, tn = (N + 7) >> 3, tiles = tm * tn;
    if (tiles == 0 || K <= 0) return;
    const int ksteps = (K + 7) >> 3;
    int S = 1;
    if (tiles < nw) {
        S = min(nw / tiles, max(1, ksteps / 4));
        S = max(1, min(S, scratch_elems / (tiles * 128)));
    }
    for (int w = warp; w < tiles * S; w += nw) {
        const int tile = w % tiles, s = w / tiles;
        const int i0 = (tile / tn) << 4, j0 = (tile % tn) << 3;
        const int ks0 = (ksteps * s) / S, ks1 = (ksteps * (s + 1)) / S;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const int ia = i0 + g, ib = i0 + g + 8, jb = j0 + g;
        for (int ks = ks0; ks < ks1; ++ks) {
            const int k0 = (ks << 3) + t, k1 = k0 + 4;
            double a[4], b[2];
            a[0] = (ia < M && k0 < K) ? A[ia * ars + k0 * acs] : 0.0;
            a[1] = (ib < M && k0 < K) ? A[ib * ars + k0 * acs] : 0.0;
            a[2] = (ia < M && k1 < K) ? A[ia * ars + k1 * acs] : 0.0;
            a[3] = (ib < M && k1 < K) ? A[ib * ars + k1 * acs] : 0.0;
            b[0] = (jb < N && k0 < K) ? B[k0 * brs + jb * bcs] : 0.0;
            b[1] = (jb < N && k1 < K) ? B[k1 * brs + jb * bcs] : 0.0;
            dmma_16x8x8(acc, a, b);
        }
        if (S == 1) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = i0 + g + ((e >> 1) << 3), j = j0 + 2 * t + (e & 1);
                if (i < M && j < N) {
                    double* c = C + i * crs + j * ccs;
                    *c = accumulate ? *c + alpha * acc[e] : alpha * acc[e];
                }
            }
        } else {
            double* p = scratch + (s * tiles + tile) * 128 + lane * 4;
#pragma unroll
            for (int e = 0; e < 4; ++e) p[e] = acc[e];
        }
    }
    if (S > 1) {
        if (nw == all) __syncthreads();
        else asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nw * 32) : "memory");
        for (int e = warp * 32 + lane; e < tiles * 128; e += nw * 32) {
            const int tile = e >> 7, ln = (e >> 2) & 31, el = e & 3;
            const int i = ((tile / tn) << 4) + (ln >> 2) + ((el >> 1) << 3);
            const int j = ((tile % tn) << 3) + 2 * (ln & 3) + (el & 1);
            double v = scratch[e];
            for (int s = 1; s < S; ++s) v += scratch[s * tiles * 128 + e];
            if (i < M && j < N) {
                double* c = C + i * crs + j * ccs;
                *c = accumulate ? *c + alpha * v : alpha * v;
            }
        }
    }
}

// Rank-k (k <= 16) update of a block in GLOBAL memory (L2): C(i,j) -= sum_k V(i,k) Z(k,j), with
// V (M x k) and Z (k x N) in shared memory: V(i,k) = V[k*ldv + i], Z(k,j) = Z[k*ldz + j],
// C(i,j) = C[j*ldc + i]. The trailing update of the big-block QR: every output tile is a
// read-modify-write of C, so each warp handles four tiles per iteration and requests their C
// values before the DMMAs — the generic loop's one-tile-at-a-time dependent load cost ~900 cycles
// per tile. Same k order per entry as cta_mm_f64.
__device__ __forceinline__ void cta_rank_update_global(int M, int N, int K, const double* V, int ldv, const double* Z,
                                                       int ldz, double* C, int ldc) {
    const int lane = threadIdx.x & 31, warp = int(threadIdx.x >> 5), nw = int(blockDim.x >> 5);
    const int g = lane >> 2, t = lane & 3;
    const int tm = (M + 15) >> 4, tn = (N + 7) >> 3, tiles = tm * tn;
    const int ksteps = (K + 7) >> 3;
    constexpr int TB = 4;
    // tiles in column-major order (consecutive tiles of a warp batch walk down the rows of one
    // 8-column strip: 64-byte segments of consecutive addresses)
    for (int w0 = warp * TB; w0 < tiles; w0 += nw * TB) {
        double acc[TB][4], cold[TB][4];
        int i0[TB], j0[TB];
#pragma unroll
        for (int b = 0; b < TB; ++b) {
            const int w = w0 + b;
            const bool on = w < tiles;
            i0[b] = on ? (w % tm) << 4 : M;  // off tiles: every predicate below fails
            j0[b] = on ? (w / tm) << 3 : N;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = i0[b] + g + ((e >> 1) << 3), j = j0[b] + 2 * t + (e & 1);
                acc[b][e] = 0.0;
                cold[b][e] = (i < M && j < N) ? C[int64_t(j) * ldc + i] : 0.0;
            }
        }
        for (int ks = 0; ks < ksteps; ++ks) {
            const int k0 = (ks << 3) + t, k1 = k0 + 4;
#pragma unroll
            for (int b = 0; b < TB; ++b) {
                const int ia = i0[b] + g, ib = ia + 8, jb = j0[b] + g;
                double a[4], bb[2];
                a[0] = (ia < M && k0 < K) ? V[k0 * ldv + ia] : 0.0;
                a[1] = (ib < M && k0 < K) ? V[k0 * ldv + ib] : 0.0;
                a[2] = (ia < M && k1 < K) ? V[k1 * ldv + ia] : 0.0;
                a[3] = (ib < M && k1 < K) ? V[k1 * ldv + ib] : 0.0;
                bb[0] = (jb < N && k0 < K) ? Z[k0 * ldz + jb] : 0.0;
                bb[1] = (jb < N && k1 < K) ? Z[k1 * ldz + jb] : 0.0;
                dmma_16x8x8(acc[b], a, bb);
            }
        }
#pragma unroll
        for (int b = 0; b < TB; ++b)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = i0[b] + g + ((e >> 1) << 3), j = j0[b] + 2 * t + (e & 1);
                if (i < M && j < N) C[int64_t(j) * ldc + i] = cold[b][e] - acc[b][e];
            }
    }
}

// E(i,j) -= sum_k V(i,k) Z(k,j) for a tall E (M x N, N <= 32) in shared memory, V (M x K, K <= 16)
// in GLOBAL memory (L2) and Z (K x N) in shared memory:
//   V(i,k) = V[k*ldv + i], Z(k,j) = Z[k*ldz + j], E(i,j) = E[j*lde + i].
// The rank-16 step of the explicit-Q kernel on big TSQR blocks. The generic cta_mm_f64 spends ~170
// instructions per 16 x 8 tile there (predicated element loads with runtime strides, once per
// tile: ncu showed the kernel issue-bound at 0.8 % FP64-pipe activity); here a warp owns a 16-row
// strip: the Z fragments of all column tiles are loaded once per call, the V fragments once per
// strip and reused by its (up to four) tiles. Same DMMA order and the same c + (-acc) update per
// entry as cta_mm_f64(alpha = -1, accumulate): bit-identical.
__device__ __forceinline__ void cta_strip_update_ga(int M, int N, int K, const double* __restrict__ V, int ldv,
                                                    const double* Z, int ldz, double* E, int lde) {
    const int lane = threadIdx.x & 31, warp = int(threadIdx.x >> 5), nw = int(blockDim.x >> 5);
    const int g = lane >> 2, t = lane & 3;
    const int tm = (M + 15) >> 4, tn = (N + 7) >> 3;
    double zb[2][4][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) {
            const int k0 = 8 * u + t, k1 = k0 + 4, jb = 8 * jt + g;
            zb[u][jt][0] = (jb < N && k0 < K) ? Z[k0 * ldz + jb] : 0.0;
            zb[u][jt][1] = (jb < N && k1 < K) ? Z[k1 * ldz + jb] : 0.0;
        }
    const bool two = K > 8;
    for (int strip = warp; strip < tm; strip += nw) {
        const int ia = (strip << 4) + g, ib = ia + 8;
        double a[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int k0 = 8 * u + t, k1 = k0 + 4;
            a[u][0] = (ia < M && k0 < K) ? V[k0 * ldv + ia] : 0.0;
            a[u][1] = (ib < M && k0 < K) ? V[k0 * ldv + ib] : 0.0;
            a[u][2] = (ia < M && k1 < K) ? V[k1 * ldv + ia] : 0.0;
            a[u][3] = (ib < M && k1 < K) ? V[k1 * ldv + ib] : 0.0;
        }
        double cold[4][4];  // the strip's E entries, requested before the DMMAs
#pragma unroll
        for (int jt = 0; jt < 4; ++jt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = (strip << 4) + g + ((e >> 1) << 3), j = 8 * jt + 2 * t + (e & 1);
                cold[jt][e] = (i < M && j < N) ? E[j * lde + i] : 0.0;
            }
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) {
            if (jt >= tn) break;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            dmma_16x8x8(acc, a[0], zb[0][jt]);
            if (two) dmma_16x8x8(acc, a[1], zb[1][jt]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = (strip << 4) + g + ((e >> 1) << 3), j = 8 * jt + 2 * t + (e & 1);
                if (i < M && j < N) E[j * lde + i] = cold[jt][e] + (-1.0) * acc[e];
            }
        }
    }
}

// Y(a,j) = sum_r V(r,a) E(r,j) for the same operands (a < M <= 16 reflector columns, j < N <= 32,
// r < K rows): V(r,a) = V[a*ldv + r] (global), E(r,j) = E[j*lde + r] (shared), Y(a,j) = Y[a*ldy + j].
// cta_mm_f64's partition exactly — (column tile, K split) per warp, the same k ranges, the partial
// tiles summed in split order through `scratch` — with contiguous-k pointers and only the last
// k-step predicated on k: bit-identical, ~3x fewer instructions.
__device__ __forceinline__ void cta_vt_e_ga(int M, int N, int K, const double* __restrict__ V, int ldv, const double* E,
                                            int lde, double* Y, int ldy, double* scratch, int scratch_elems) {
    const int lane = threadIdx.x & 31, warp = int(threadIdx.x >> 5), nw = int(blockDim.x >> 5);
    const int g = lane >> 2, t = lane & 3;
    const int tn = (N + 7) >> 3, tiles = tn;  // M <= 16: one tile row
    if (tiles == 0 || K <= 0) return;
    const int ksteps = (K + 7) >> 3;
    int S = 1;
    if (tiles < nw) {
        S = min(nw / tiles, max(1, ksteps / 4));
        S = max(1, min(S, scratch_elems / (tiles * 128)));
    }
    const int kfull = K >> 3;  // k-steps with all 8 k inside [0, K)
    for (int w = warp; w < tiles * S; w += nw) {
        const int tile = w % tiles, s = w / tiles;
        const int jb = (tile << 3) + g;
        const int ks0 = (ksteps * s) / S, ks1 = (ksteps * (s + 1)) / S;
        const bool va = g < M, vb = g + 8 < M, vj = jb < N;
        const double* pa0 = V + (va ? g : 0) * ldv + t;
        const double* pa1 = V + (vb ? g + 8 : 0) * ldv + t;
        const double* pb = E + (vj ? jb : 0) * lde + t;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const int ksm = min(ks1, kfull);
        int ks = ks0;
        constexpr int KB = 5;  // k-steps whose V fragments (L2) are requested together
        for (; ks + KB <= ksm; ks += KB) {
            double a[KB][4];
#pragma unroll
            for (int u = 0; u < KB; ++u) {
                const int k = (ks + u) << 3;
                a[u][0] = pa0[k];
                a[u][1] = pa1[k];
                a[u][2] = pa0[k + 4];
                a[u][3] = pa1[k + 4];
            }
#pragma unroll
            for (int u = 0; u < KB; ++u) {
                const int k = (ks + u) << 3;
                double b[2] = {pb[k], pb[k + 4]};
                if (!va) a[u][0] = a[u][2] = 0.0;
                if (!vb) a[u][1] = a[u][3] = 0.0;
                if (!vj) b[0] = b[1] = 0.0;
                dmma_16x8x8(acc, a[u], b);
            }
        }
        for (; ks < ksm; ++ks) {
            const int k = ks << 3;
            double a[4] = {pa0[k], pa1[k], pa0[k + 4], pa1[k + 4]}, b[2] = {pb[k], pb[k + 4]};
            if (!va) a[0] = a[2] = 0.0;
            if (!vb) a[1] = a[3] = 0.0;
            if (!vj) b[0] = b[1] = 0.0;
            dmma_16x8x8(acc, a, b);
        }
        for (; ks < ks1; ++ks) {  // the ragged last k-step
            const int k0 = (ks << 3) + t, k1 = k0 + 4;
            double a[4], b[2];
            a[0] = (va && k0 < K) ? pa0[ks << 3] : 0.0;
            a[1] = (vb && k0 < K) ? pa1[ks << 3] : 0.0;
            a[2] = (va && k1 < K) ? pa0[(ks << 3) + 4] : 0.0;
            a[3] = (vb && k1 < K) ? pa1[(ks << 3) + 4] : 0.0;
            b[0] = (vj && k0 < K) ? pb[ks << 3] : 0.0;
            b[1] = (vj && k1 < K) ? pb[(ks << 3) + 4] : 0.0;
            dmma_16x8x8(acc, a, b);
        }
        if (S == 1) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = g + ((e >> 1) << 3), j = (tile << 3) + 2 * t + (e & 1);
                if (i < M && j < N) Y[i * ldy + j] = 1.0 * acc[e];
            }
        } else {
            double* p = scratch + (s * tiles + tile) * 128 + lane * 4;
#pragma unroll
            for (int e = 0; e < 4; ++e) p[e] = acc[e];
        }
    }
    if (S > 1) {
        __syncthreads();
        for (int e = warp * 32 + lane; e < tiles * 128; e += nw * 32) {
            const int tile = e >> 7, ln = (e >> 2) & 31, el = e & 3;
            const int i = (ln >> 2) + ((el >> 1) << 3);
            const int j = (tile << 3) + 2 * (ln & 3) + (el & 1);
            double v = scratch[e];
            for (int s = 1; s < S; ++s) v += scratch[s * tiles * 128 + e];
            if (i < M && j < N) Y[i * ldy + j] = 1.0 * v;
        }
    }
}

// Same contract for any T on the CUDA cores (fp32 path; small fp64 shapes).
template <typename T>
__device__ __forceinline__ void cta_mm_simt(int M, int N, int K, const T* A, int ars, int acs, const T* B, int brs,
                                            int bcs, T* C, int crs, int ccs, T alpha, bool accumulate, T* scratch,
                                            int scratch_elems) {
    cta_gemm<2, 2, T>(
        M, N, K, [=] __device__(int i, int k) { return A[i * ars + k * acs]; },
        [=] __device__(int k, int j) { return B[k * brs + j * bcs]; },
        [=] __device__(int i, int j, T v) {
            T* c = C + i * crs + j * ccs;
            *c = accumulate ? *c + alpha * v : alpha * v;
        },
        scratch, scratch_elems);
}

__device__ __forceinline__ void cta_mm(int M, int N, int K, const double* A, int ars, int acs, const double* B, int brs,
                                       int bcs, double* C, int crs, int ccs, double alpha, bool accumulate,
                                       double* scratch, int scratch_elems, int warp0 = 0, int nwarps = -1) {
    cta_mm_f64(M, N, K, A, ars, acs, B, brs, bcs, C, crs, ccs, alpha, accumulate, scratch, scratch_elems, warp0, nwarps);
}
__device__ __forceinline__ void cta_mm(int M, int N, int K, const float* A, int ars, int acs, const float* B, int brs,
                                       int bcs, float* C, int crs, int ccs, float alpha, bool accumulate,
                                       float* scratch, int scratch_elems) {
    cta_mm_simt<float>(M, N, K, A, ars, acs, B, brs, bcs, C, crs, ccs, alpha, accumulate, scratch, scratch_elems);
}

// Forward compact-WY T factor (LAPACK dlarft convention): H_0 H_1 ... H_{k-1} = I - V T V^T with
// T upper triangular, T(j,j) = beta_j and T(0:j, j) = -beta_j T(0:j, 0:j) G(0:j, j), where
// G(a,b) = v_a^T v_b (a < b) is given (ldg). One warp. For k <= 16 lane a owns row a of T in
// registers (see below); wider panels use the generic shared-memory loop.
template <typename T>
__device__ __forceinline__ void warp_larft(int k, const T* G, int ldg, const T* beta, T* Tm, int ldt) {
    const int lane = threadIdx.x & 31;
    if (k <= 16) {
        // Lane a keeps row a of T in registers; the loops are fully unrolled so every register
        // index is static, and column b of G is read as broadcast loads (no dependent smem chain).
        // Row a is zero left of the diagonal, so the sum needs no predicate; columns b >= k are
        // computed from clamped (finite or not, never stored) entries and discarded.
        const int a = lane;
        T row[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) row[c] = T(0);
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const T bb = beta[b < k ? b : k - 1];
            // Branch-free: the newest entry row[b-1] enters last, so the per-column critical path is
            // two dependent FMAs; fma(-bb, s, 0) rounds exactly like -bb * s.
            T p0 = 0, p1 = 0;
#pragma unroll
            for (int c = 0; c + 1 < b; ++c) {
                const T gv = G[c * ldg + b];
                if (c & 1) p1 = fma(row[c], gv, p1);
                else p0 = fma(row[c], gv, p0);
            }
            const T s = b > 0 ? fma(row[b - 1], G[(b - 1) * ldg + b], p0 + p1) : T(0);
            const T coef = a < b ? -bb : T(0), diag = a == b ? bb : T(0);
            row[b] = fma(coef, s, diag);
        }
        if (a < k) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < k) Tm[a * ldt + c] = row[c];
        }
        __syncwarp();
        return;
    }
    for (int b = 0; b < k; ++b) {
        const T bb = beta[b];
        for (int a = lane; a < k; a += 32) {
            if (a < b) {
                T s = 0;
                for (int c = a; c < b; ++c) s += Tm[a * ldt + c] * G[c * ldg + b];
                Tm[a * ldt + b] = -bb * s;
            } else {
                Tm[a * ldt + b] = a == b ? bb : T(0);
            }
        }
        __syncwarp();
    }
}

}  // namespace coru_gpu
