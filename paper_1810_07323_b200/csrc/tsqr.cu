// TSQR with CTA-local Householder panels and an R-factor reduction tree.
//
// Replaces householder_qr (proj/include/coru/qr.hpp:85-99) at corutv.hpp:59-60 (QR of the
// sketches c1, c2). Every block runs the reference's unblocked reflector recipe —
// make_reflector (qr.hpp:32-45: mu = ||x||, v0 = x0 - mu or -sigma/(x0+mu), beta = 2v0^2/(sigma+v0^2),
// v scaled by 1/v0, sigma == 0 leaves the column untouched) and apply_reflector (qr.hpp:49-57) —
// so every R on the tree has diag >= 0 and the explicit Q equals the reference's Q up to rounding
// (the QR with positive diagonal is unique for full-rank input).
//
// Factor kernel: one CTA per block; the block sits column-major in shared memory (or in L2 for
// wide d). Column c is owned by warp c % NW for the whole factorisation, so the only
// cross-warp dependency is "reflector j is ready", published through a per-column acquire/
// release flag in shared memory — no __syncthreads in the column loop. The owner of column
// j+1 applies H_j to it first and publishes reflector j+1 before touching its other columns
// (look-ahead), which keeps the critical path at one column update + one norm per step.
//
// Q kernel: applies the stored reflectors backwards (accumulate_q order, qr.hpp:60-72) onto
// [Q_above block; 0]; columns are independent, so warps never synchronise.
//
// Two implementations share the tree: the blocked one below (shared-memory block, panels +
// compact WY) whenever a block of > 1.25 d rows fits shared memory, and the "wide" one (the
// unblocked column pipeline, working block in L2) for sketch widths too wide for that.
#include <cstdlib>
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include <type_traits>
#include "cta_blas.cuh"
#include "tsqr.cuh"

namespace coru_gpu {

#ifdef CORU_QR_PROFILE
__device__ long long g_qrg_phase[12];  // k_qr_blocked_g, block 0: load, chain, gram, larft, Y, Z, update, export, total
#define QRG_T(v) long long v = qrp_clock_fwd()
// the clock is read in the same asm statement as a CTA barrier, so ptxas cannot hoist it above the wait
#define QRG_ADD(i, v) { long long n_; asm volatile("bar.sync 0;\n\tmov.u64 %0, %%clock64;" : "=l"(n_)::"memory"); \
                        if (threadIdx.x == 0 && blockIdx.x == 0) g_qrg_phase[i] += n_ - v; v = n_; }
__device__ __forceinline__ long long qrp_clock_fwd() { long long v; asm volatile("mov.u64 %0, %%clock64;" : "=l"(v)::"memory"); return v; }
__device__ long long g_qr_phase[12];
__device__ long long g_qr_tl[3 * 256];  // block 0 chain timeline: arrive / wake / build-start per column  // cycles of block 0: load, panel chains, T factors, trailing, export
__device__ __forceinline__ long long qrp_clock() {
    long long v;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(v)::"memory");
    return v;
}
#define QRP_T(v) long long v = qrp_clock()
#define QRP_NS(v) unsigned long long v; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#define QRP_NSADD(i, t0) if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned long long t1_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1_)); g_qr_phase[i] += t1_ - (t0); }
// per-thread register accumulators; block 0 / thread 0 flushes them once at the end
#define QRP_DECL long long qrp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define QRP_ADD(i, t0) qrp_acc[i] += qrp_clock() - (t0)
#define QRP_TL(k, j) if (blockIdx.x == 0 && lane == 0) g_qr_tl[(k) * 256 + (j)] = qrp_clock()
#define QRP_FLUSH if (threadIdx.x == 0 && blockIdx.x == 0) for (int i_ = 0; i_ < 8; ++i_) g_qr_phase[i_] += qrp_acc[i_]
// k_qr_reg timeline: per step, cycles of [v load, apply, build, barrier] summed for warp 0 and for
// the building warp (clock read made dependent on the phase's last result)
__device__ long long g_qr_reg_ph[8];
#define QRR_CLK(v, dep) long long v; asm volatile("mov.u64 %0, %%clock64;" : "=l"(v) : "d"(double(dep)) : "memory")
#define QRR_ADD(i, dt) if (blockIdx.x == 0 && lane == 0) atomicAdd((unsigned long long*)&g_qr_reg_ph[i], (unsigned long long)(dt))
#else
#define QRP_T(v)
#define QRP_ADD(i, t0)
#define QRP_NS(v)
#define QRP_NSADD(i, t0)
#define QRP_DECL
#define QRP_TL(k, j)
#define QRP_FLUSH
#define QRG_T(v)
#define QRG_ADD(i, v)
#define QRR_CLK(v, dep)
#define QRR_ADD(i, dt)
#endif

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ int ld_acquire_flag(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_flag(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T tsqrt(T x);
template <>
__device__ __forceinline__ double tsqrt<double>(double x) { return sqrt(x); }
template <>
__device__ __forceinline__ float tsqrt<float>(float x) { return sqrtf(x); }

// Build reflector for column j of the column-major block W (ld ldw, rb rows); one warp.
// Returns beta (also stored), column scaled in place, W[j][j] = mu.  (qr.hpp:32-45)
template <typename T>
__device__ __forceinline__ T warp_make_reflector(T* col, int rb, int j, int lane) {
    T sig = 0;
    for (int i = j + 1 + lane; i < rb; i += 32) sig += col[i] * col[i];
    sig = warp_sum(sig);
    const T x0 = col[j];
    if (sig == T(0)) return T(0);
    T mu, v0, beta, rv;
    reflector_scalars(x0, sig, mu, v0, beta, rv);
    for (int i = j + 1 + lane; i < rb; i += 32) col[i] *= rv;
    __syncwarp();
    if (lane == 0) col[j] = mu;
    __syncwarp();
    return beta;
}

// (I - beta v v^T) col, v = [1; vcol[j+1:rb]]   (qr.hpp:49-57)
template <typename T>
__device__ __forceinline__ void warp_apply_reflector(const T* vcol, T beta, int rb, int j, T* col, int lane) {
    if (beta == T(0)) return;
    T s = 0;
    for (int i = j + 1 + lane; i < rb; i += 32) s += vcol[i] * col[i];
    s = warp_sum(s);
    s += col[j];
    s *= beta;
    for (int i = j + 1 + lane; i < rb; i += 32) col[i] -= s * vcol[i];
    __syncwarp();
    if (lane == 0) col[j] -= s;
    __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_hh_factor(const T* __restrict__ X, int64_t ldx, int64_t rows, int nb,
                                                        int d, T* __restrict__ V, int ldv, T* __restrict__ betas,
                                                        T* __restrict__ Rout, int ldr, int use_smem, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    int* flags = reinterpret_cast<int*>(smem_raw);                 // d ints
    T* sbeta = reinterpret_cast<T*>(smem_raw + ((d * 4 + 15) / 16) * 16);  // d T
    T* W;
    int ldw;
    T* Vb = V + int64_t(b) * d * ldv;
    if (use_smem) {
        W = sbeta + ((d + 1) / 2) * 2;
        ldw = rb | 1;  // odd column stride: conflict-free transposing stores
    } else {
        W = Vb;
        ldw = ldv;
    }
    for (int c = tid; c < d; c += kThreads) flags[c] = 0;
    // Load rows [r0, r1) (row-major) into column-major W.
    for (int64_t e = tid; e < int64_t(rb) * d; e += kThreads) {
        const int r = int(e / d), c = int(e % d);
        W[int64_t(c) * ldw + r] = X[(r0 + r) * ldx + c];
    }
    __syncthreads();

    // Look-ahead column pipeline.
    if (warp == 0 % kWarps) {
        const T beta0 = warp_make_reflector(W, rb, 0, lane);
        if (lane == 0) {
            sbeta[0] = beta0;
            st_release_flag(&flags[0], 1);
        }
        __syncwarp();
    }
    for (int j = 0; j < d; ++j) {
        if (lane == 0)
            while (ld_acquire_flag(&flags[j]) == 0) {
            }
        __syncwarp();
        const T beta = *reinterpret_cast<volatile T*>(&sbeta[j]);
        const T* vcol = W + int64_t(j) * ldw;
        int c = j + 1 + ((warp - (j + 1)) % kWarps + kWarps) % kWarps;  // first column > j owned by me
        for (; c < d; c += kWarps) {
            T* col = W + int64_t(c) * ldw;
            warp_apply_reflector(vcol, beta, rb, j, col, lane);
            if (c == j + 1) {
                const T bn = warp_make_reflector(col, rb, c, lane);
                if (lane == 0) {
                    sbeta[c] = bn;
                    st_release_flag(&flags[c], 1);
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();

    // R (upper triangle, exact zeros below; qr.hpp:74-79) -> rows [b*d, (b+1)*d) of Rout.
    for (int e = tid; e < d * d; e += kThreads) {
        const int r = e / d, c = e % d;
        Rout[(int64_t(b) * d + r) * ldr + c] = (r <= c) ? W[int64_t(c) * ldw + r] : T(0);
    }
    for (int c = tid; c < d; c += kThreads) betas[int64_t(b) * d + c] = sbeta[c];
    if (use_smem) {
        for (int64_t e = tid; e < int64_t(rb) * d; e += kThreads) {
            const int c = int(e / rb), r = int(e % rb);
            Vb[int64_t(c) * ldv + r] = W[int64_t(c) * ldw + r];
        }
    }
}

// Q block b = H_b · [Qin[b*d:(b+1)*d, :]; 0]   (Qin null => identity), written to Qout rows [r0, r1).
template <typename T>
__global__ void __launch_bounds__(kThreads) k_hh_form_q(const T* __restrict__ Qin, int ldqin, int64_t rows, int nb,
                                                        int d, const T* __restrict__ V, int ldv,
                                                        const T* __restrict__ betas, T* __restrict__ Qout,
                                                        int64_t ldqout, T* __restrict__ gscratch, int use_smem, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T* Vb = V + int64_t(b) * d * ldv;
    const T* bb = betas + int64_t(b) * d;
    T* E;
    int lde;
    if (use_smem) {
        E = reinterpret_cast<T*>(smem_raw);
        lde = rb | 1;
    } else {
        E = gscratch + int64_t(b) * d * ldv;
        lde = ldv;
    }
    for (int64_t e = tid; e < int64_t(rb) * d; e += kThreads) {
        const int r = int(e / d), c = int(e % d);
        T x = T(0);
        if (r < d) x = Qin ? Qin[(int64_t(b) * d + r) * ldqin + c] : T(r == c ? 1 : 0);
        E[int64_t(c) * lde + r] = x;
    }
    __syncthreads();
    for (int c = warp; c < d; c += kWarps) {
        T* col = E + int64_t(c) * lde;
        for (int j = d - 1; j >= 0; --j) {
            const T beta = bb[j];
            if (beta == T(0)) continue;
            const T* vcol = Vb + int64_t(j) * ldv;
            T s = 0;
            for (int i = j + 1 + lane; i < rb; i += 32) s += __ldg(&vcol[i]) * col[i];
            s = warp_sum(s);
            s += col[j];
            s *= beta;
            for (int i = j + 1 + lane; i < rb; i += 32) col[i] -= s * __ldg(&vcol[i]);
            __syncwarp();
            if (lane == 0) col[j] -= s;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int64_t e = tid; e < int64_t(rb) * d; e += kThreads) {
        const int r = int(e / d), c = int(e % d);
        Qout[(r0 + r) * ldqout + c] = E[int64_t(c) * lde + r];
    }
}


// ============================================================================================
// Blocked path (the block fits shared memory). Panels of kNB columns are factored with the column
// pipeline held in registers (one warp per panel column, a column = kRPL values per lane), the
// "reflector j ready" hand-off going through named hardware barriers (bar.arrive by the builder,
// bar.sync by the later panel warps: no spinning). The panel's explicit reflectors V_p and its
// compact-WY factor T_p (H_p0...H_p0+nb-1 = I - V_p T_p V_p^T, dlarft convention) then update the
// trailing columns with three DMMA GEMMs, C <- C - V_p T_p^T (V_p^T C). The per-panel T_p are kept,
// so Q is formed panel by panel (in reverse) with the same GEMM shape.
// ============================================================================================
constexpr int kBThreads = 512;
constexpr int kNB = 16;       // panel width == warps that own a panel column
constexpr int kRPL = 8;       // rows per lane held in registers: blocks of <= 256 rows
constexpr int kMaxRowsBlocked = 32 * kRPL;
constexpr int kGemmScratch = 2048;
constexpr int kQChunk = 32;   // Q columns formed per pass

__host__ __device__ inline int ld_mod(int rows, int residue) {
    // smallest ld >= rows with ld % 16 == residue (bank-friendly fragment strides for 8-byte data)
    int ld = rows;
    while (ld % 16 != residue) ++ld;
    return ld;
}
__host__ __device__ inline int npanels(int d) { return (d + kNB - 1) / kNB; }

__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <typename T>
struct BlockedSmem {
    int d, ldw, ldvp;
    T *W, *Vp, *beta, *Gp, *Tp, *Y, *Z, *scratch;
    __device__ BlockedSmem(unsigned char* raw, int d_, int rb) : d(d_), ldw(ld_mod(rb, 4)), ldvp(ld_mod(rb, 8)) {
        T* p = reinterpret_cast<T*>(raw);
        W = p;
        p += size_t(d) * ldw;
        Vp = p;
        p += size_t(kNB) * ldvp;
        beta = p;
        p += d + (d & 1);
        Gp = p;
        p += kNB * kNB;
        Tp = p;
        p += kNB * kNB;
        Y = p;
        p += size_t(kNB) * d;
        Z = p;
        p += size_t(kNB) * d;
        scratch = p;
    }
    static size_t bytes(int d, int rb, size_t eb) {
        return (size_t(d) * ld_mod(rb, 4) + size_t(kNB) * ld_mod(rb, 8) + d + (d & 1) + 2 * kNB * kNB +
                2 * size_t(kNB) * d + kGemmScratch) *
               eb;
    }
};

template <typename T>
__global__ void __launch_bounds__(kBThreads, 1)
    k_qr_blocked(const T* __restrict__ X, int64_t ldx, int64_t rows, int nb, int d, T* __restrict__ V, int ldv,
                 T* __restrict__ betas, T* __restrict__ Tg, T* __restrict__ Rout, int ldr, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    BlockedSmem<T> S(smem_raw, d, rb);
    T* W = S.W;
    const int ldw = S.ldw, ldvp = S.ldvp;
    T* Tb = Tg + int64_t(b) * npanels(d) * kNB * kNB;  // this block's panel T factors

    QRP_DECL;
    QRP_NS(ns_all);
    QRP_T(t_all);
    QRP_T(t_load);
    // Load rows [r0, r1) (row-major, coalesced along columns) into column-major W; four rows in
    // flight per warp for memory-level parallelism.
    for (int cb = 0; cb < d; cb += 128)
        for (int r = warp * 4; r < rb; r += (kBThreads / 32) * 4) {
            T v[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int c = cb + lane + 32 * h;
                    v[q][h] = (r + q < rb && c < d) ? X[(r0 + r + q) * ldx + c] : T(0);
                }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int c = cb + lane + 32 * h;
                    if (r + q < rb && c < d) W[c * ldw + r + q] = v[q][h];
                }
        }
    __syncthreads();

    QRP_ADD(0, t_load);
    for (int p0 = 0, pi = 0; p0 < d; p0 += kNB, ++pi) {
        const int nbp = min(kNB, d - p0);
        QRP_T(t_chain);
        // ---- panel factorisation: warp w owns column p0 + w; rows >= p0 in registers ----
        if (warp < nbp) {
            const int c = p0 + warp;
            T x[kRPL];
#pragma unroll
            for (int u = 0; u < kRPL; ++u) {
                const int r = lane + 32 * u;
                x[u] = (r >= p0 && r < rb) ? W[c * ldw + r] : T(0);
            }
            for (int jj = 0; jj <= warp; ++jj) {
                const int j = p0 + jj;
                const int bar = 1 + jj, cnt = 32 * (nbp - jj);
                if (jj < warp) {
                    // apply H_j (built by warp jj) to my column   (apply_reflector, qr.hpp:49-57)
                    named_bar_sync(bar, cnt);
                    if (jj + 1 == warp) QRP_TL(1, j + 1);
                    const T bj = S.beta[j];
                    if (bj == T(0)) continue;
                    const T* vj = S.Vp + jj * ldvp;
                    T v[kRPL], pr[kRPL];
#pragma unroll
                    for (int u = 0; u < kRPL; ++u) {
                        const int r = lane + 32 * u;
                        v[u] = r < rb ? vj[r] : T(0);
                        pr[u] = v[u] * x[u];
                    }
                    // pairwise (tree) sum: short dependency chain on the critical path
#pragma unroll
                    for (int h = kRPL / 2; h > 0; h >>= 1)
#pragma unroll
                        for (int u = 0; u < h; ++u) pr[u] += pr[u + h];
                    const T s = warp_sum(pr[0]) * bj;
#pragma unroll
                    for (int u = 0; u < kRPL; ++u) x[u] -= s * v[u];
                } else {
                    // build reflector j from my column   (make_reflector, qr.hpp:32-45)
                    QRP_TL(2, j);
                    T sq[kRPL];
#pragma unroll
                    for (int u = 0; u < kRPL; ++u) {
                        const int r = lane + 32 * u;
                        sq[u] = r > j ? x[u] * x[u] : T(0);
                        if (r == j) W[c * ldw + j] = x[u];  // x0 through smem: no dynamic register index
                    }
#pragma unroll
                    for (int h = kRPL / 2; h > 0; h >>= 1)
#pragma unroll
                        for (int u = 0; u < h; ++u) sq[u] += sq[u + h];
                    const T sig = warp_sum(sq[0]);
                    __syncwarp();
                    const T x0 = W[c * ldw + j];
                    T bj = 0;
                    if (sig != T(0)) {
                        // v = x / v0 (qr.hpp:42) as x · (1/v0); short-latency scalars (common.cuh)
                        T mu, v0, rv;
                        reflector_scalars(x0, sig, mu, v0, bj, rv);
#pragma unroll
                        for (int u = 0; u < kRPL; ++u) {
                            const int r = lane + 32 * u;
                            x[u] = r > j ? x[u] * rv : (r == j ? mu : x[u]);
                        }
                    }
                    T* vj = S.Vp + jj * ldvp;
#pragma unroll
                    for (int u = 0; u < kRPL; ++u) {
                        const int r = lane + 32 * u;
                        if (r >= p0 && r < rb) W[c * ldw + r] = x[u];
                        // explicit reflector: 0 above j, 1 at j, v below (0 past rb and in the padding)
                        if (r < ldvp) vj[r] = (r > j && r < rb) ? x[u] : (r == j ? T(1) : T(0));
                    }
                    if (lane == 0) S.beta[j] = bj;
                    QRP_TL(0, j);
                    if (jj + 1 < nbp) named_bar_arrive(bar, cnt);
                }
            }
        }
        __syncthreads();
        QRP_ADD(1, t_chain);
        QRP_T(t_tf);
        const int K = rb - p0;
        const int c0 = p0 + nbp, nc = d - c0;
        T* C = W + c0 * ldw + p0;
#ifdef CORU_ABL_CHAIN_ONLY  // tooling ablation: the panel chains alone (wrong results)
        continue;
#endif
        // ---- panel T factor: G = V_p^T V_p, T_p by the forward recurrence ----
        cta_mm(nbp, nbp, K, S.Vp + p0, ldvp, 1, S.Vp + p0, 1, ldvp, S.Gp, kNB, 1, T(1), false, S.scratch, kGemmScratch);
        QRP_ADD(6, t_tf);
        __syncthreads();
        QRP_ADD(5, t_tf);
        // The recurrence (one warp) overlaps Y = V_p^T C on the other warps (fp64 tensor path).
        constexpr bool kOverlap = sizeof(T) == 8;
        if (warp == 0) {
            warp_larft<T>(nbp, S.Gp, kNB, S.beta + p0, S.Tp, kNB);
            T* Tpg = Tb + pi * kNB * kNB;
            for (int e = lane; e < kNB * kNB; e += 32) Tpg[e] = S.Tp[e];
        } else if constexpr (kOverlap) {
            if (nc > 0)
                cta_mm_f64(nbp, nc, K, reinterpret_cast<const double*>(S.Vp + p0), ldvp, 1,
                           reinterpret_cast<const double*>(C), 1, ldw, reinterpret_cast<double*>(S.Y), d, 1, 1.0,
                           false, reinterpret_cast<double*>(S.scratch), kGemmScratch, 1, kBThreads / 32 - 1, 15);
        }
        __syncthreads();
        QRP_ADD(2, t_tf);
        QRP_T(t_tr);
        // ---- trailing update of columns [p0+nbp, d): C <- C - V_p T_p^T (V_p^T C), rows >= p0 ----
#ifdef CORU_ABL_NO_TRAIL  // tooling ablation: no trailing update (wrong results)
        if (false) {
#else
        if (nc > 0) {
#endif
            if constexpr (!kOverlap) {
                cta_mm(nbp, nc, K, S.Vp + p0, ldvp, 1, C, 1, ldw, S.Y, d, 1, T(1), false, S.scratch, kGemmScratch);
                __syncthreads();
            }
            cta_mm(nbp, nc, nbp, S.Tp, 1, kNB, S.Y, d, 1, S.Z, d, 1, T(1), false, S.scratch, kGemmScratch);
            __syncthreads();
            cta_mm(K, nc, nbp, S.Vp + p0, 1, ldvp, S.Z, d, 1, C, 1, ldw, T(-1), true, S.scratch, kGemmScratch);
            __syncthreads();
        }
        QRP_ADD(3, t_tr);
    }

    QRP_T(t_exp);
    // R (upper, exact zeros below) -> Rout rows [b*d, (b+1)*d); reflectors and betas to global.
    for (int e = tid; e < d * d; e += kBThreads) {
        const int r = e / d, c = e % d;
        Rout[(int64_t(b) * d + r) * ldr + c] = (r <= c) ? W[c * ldw + r] : T(0);
    }
    for (int c = tid; c < d; c += kBThreads) betas[int64_t(b) * d + c] = S.beta[c];
    // explicit reflectors (0 above the diagonal, 1 on it) for the Q kernel
    T* Vb = V + int64_t(b) * d * ldv;
    for (int c = warp; c < d; c += kBThreads / 32)
        for (int r = lane; r < rb; r += 32) Vb[int64_t(c) * ldv + r] = r > c ? W[c * ldw + r] : T(r == c ? 1 : 0);
    QRP_ADD(4, t_exp);
    QRP_ADD(7, t_all);
    QRP_FLUSH;
    QRP_NSADD(8, ns_all);
}

// Same algorithm with the working block in global memory (L2) — blocks too tall or too wide for
// shared memory (wide sketches, e.g. d = 220 fp64 or d = 520 fp32). The panel columns are
// updated in place in L2 (four independent loads in flight per lane), the panel reflectors and
// all small factors stay in shared memory, and the trailing update is the same three CTA GEMMs.
template <typename T>
struct BigSmem {
    int ldvp;
    T *Vp, *beta, *Gp, *Tp, *Y, *Z, *scratch;
    // reflector slots are read in whole 128-row chunks by the register panels: zero-padded past rb
    __device__ BigSmem(unsigned char* raw, int d, int rb) : ldvp(ld_mod(rb + 128, 8)) {
        T* p = reinterpret_cast<T*>(raw);
        Vp = p;
        p += size_t(kNB) * ldvp;
        beta = p;
        p += d + (d & 1);
        Gp = p;
        p += kNB * kNB;
        Tp = p;
        p += kNB * kNB;
        Y = p;
        p += size_t(kNB) * d;
        Z = p;
        p += size_t(kNB) * d;
        scratch = p;
    }
    static size_t bytes(int d, int rb, size_t eb) {
        return (size_t(kNB) * ld_mod(rb + 128, 8) + d + (d & 1) + 2 * kNB * kNB + 2 * size_t(kNB) * d + kGemmScratch) * eb;
    }
};

template <typename T>
__global__ void __launch_bounds__(kBThreads, 1)
    k_qr_blocked_g(const T* __restrict__ X, int64_t ldx, int64_t rows, int nb, int d, T* __restrict__ V, int ldv,
                   T* __restrict__ betas, T* __restrict__ Tg, T* __restrict__ Rout, int ldr, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    BigSmem<T> S(smem_raw, d, rb);
    const int ldvp = S.ldvp;
    T* W = V + int64_t(b) * d * ldv;  // column-major working block (ld = ldv) in global memory
    T* Tb = Tg + int64_t(b) * npanels(d) * kNB * kNB;
    QRG_T(tq);
    // Rows [r0, r1) of X (row-major) -> column-major working block W, transposed through shared memory
    // (the reflector slots are free now): 64-row chunks read along the rows, written along the
    // columns, both coalesced (the direct transposing store touched one line per element).
    {
        // chunk rows: up to 64, fewer when d columns of them would not fit the kNB·ldvp slots
        const int kLR = min(64, (kNB * ldvp) / d - 1), kLLd = kLR + 1;
        T* stage = S.Vp;
        for (int rc = 0; rc < rb; rc += kLR) {
            const int nr = min(kLR, rb - rc);
            for (int e = tid; e < nr * d; e += kBThreads) {
                const int r = e / d, c = e % d;
                stage[c * kLLd + r] = X[(r0 + rc + r) * ldx + c];
            }
            __syncthreads();
            for (int e = tid; e < d * kLR; e += kBThreads) {
                const int c = e / kLR, r = e % kLR;
                if (r < nr) W[int64_t(c) * ldv + rc + r] = stage[c * kLLd + r];
            }
            __syncthreads();
        }
    }
    __syncthreads();
    QRG_ADD(0, tq);

    // Blocks of up to 32·kGRPL rows keep each panel column in REGISTERS while the panel is factored
    // (lane l holds rows l, l+32, ...): the d sequential reflector steps then run at shared-memory
    // latency (the reflectors Vp) instead of one L2 round trip per read-modify-write of the column
    // (~8 us per column step before: 4 levels x ~900 us at C3). Taller blocks use the in-place path.
    constexpr int kGRPL = sizeof(T) == 8 ? 28 : 56;  // 56 registers of column per lane
    const bool reg_panel = rb <= 32 * kGRPL;
    for (int p0 = 0, pi = 0; p0 < d; p0 += kNB, ++pi) {
        const int nbp = min(kNB, d - p0);
        if (warp < nbp && reg_panel) {
            // Register layout of my column for this panel: `xs` = the 32-row block that holds the
            // panel's diagonal rows (one row per lane; rows above the diagonal are final R entries
            // and are masked by the explicit zeros of the reflectors), x[] = the rows after it in
            // chunks of 4 x 32 — every loop over them is predicate-free (reflector slots are
            // zero-padded past rb), with one uniform test per chunk.
            const int c = p0 + warp;
            T* col = W + int64_t(c) * ldv;
            const int hb = (p0 >> 5) << 5, tb = hb + 32;     // head block / first tail row
            const int nt4 = (max(rb - tb, 0) + 127) >> 7;    // live tail chunks
            const int rh = hb + lane;
            T xs = (rh >= p0 && rh < rb) ? col[rh] : T(0);
            T x[kGRPL];
#pragma unroll
            for (int t4 = 0; t4 < kGRPL / 4; ++t4)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int r = tb + 32 * (4 * t4 + q4) + lane;
                    x[4 * t4 + q4] = (t4 < nt4 && r < rb) ? col[r] : T(0);
                }
            for (int jj = 0; jj <= warp; ++jj) {
                const int j = p0 + jj, jl = j - hb;
                const int bar = 1 + jj, cnt = 32 * (nbp - jj);
                if (jj < warp) {
                    // apply H_j (built by warp jj) to my column   (apply_reflector, qr.hpp:49-57)
                    named_bar_sync(bar, cnt);
                    const T bj = S.beta[j];
                    if (bj == T(0)) continue;
                    const T* vj = S.Vp + jj * ldvp;
                    const T vh = vj[rh];
                    const T* vt = vj + tb + lane;
                    T s0 = vh * xs, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
                    for (int t4 = 0; t4 < kGRPL / 4; ++t4)
                        if (t4 < nt4) {
                            s0 += vt[128 * t4] * x[4 * t4];
                            s1 += vt[128 * t4 + 32] * x[4 * t4 + 1];
                            s2 += vt[128 * t4 + 64] * x[4 * t4 + 2];
                            s3 += vt[128 * t4 + 96] * x[4 * t4 + 3];
                        }
                    const T s = warp_sum((s0 + s1) + (s2 + s3)) * bj;
                    xs -= s * vh;
#pragma unroll
                    for (int t4 = 0; t4 < kGRPL / 4; ++t4)
                        if (t4 < nt4) {
                            x[4 * t4] -= s * vt[128 * t4];
                            x[4 * t4 + 1] -= s * vt[128 * t4 + 32];
                            x[4 * t4 + 2] -= s * vt[128 * t4 + 64];
                            x[4 * t4 + 3] -= s * vt[128 * t4 + 96];
                        }
                } else {
                    // build reflector j from my column   (make_reflector, qr.hpp:32-45)
                    T q0 = lane > jl ? xs * xs : T(0), q1 = 0, q2 = 0, q3 = 0;
#pragma unroll
                    for (int t4 = 0; t4 < kGRPL / 4; ++t4)
                        if (t4 < nt4) {
                            q0 += x[4 * t4] * x[4 * t4];
                            q1 += x[4 * t4 + 1] * x[4 * t4 + 1];
                            q2 += x[4 * t4 + 2] * x[4 * t4 + 2];
                            q3 += x[4 * t4 + 3] * x[4 * t4 + 3];
                        }
                    const T sig = warp_sum((q0 + q1) + (q2 + q3));
                    const T x0 = __shfl_sync(0xffffffffu, xs, jl);
                    T bj = 0;
                    if (sig != T(0)) {
                        T mu, v0, rv;
                        reflector_scalars(x0, sig, mu, v0, bj, rv);
                        xs = lane > jl ? xs * rv : (lane == jl ? mu : xs);
#pragma unroll
                        for (int t4 = 0; t4 < kGRPL / 4; ++t4)
                            if (t4 < nt4) {
                                x[4 * t4] *= rv;
                                x[4 * t4 + 1] *= rv;
                                x[4 * t4 + 2] *= rv;
                                x[4 * t4 + 3] *= rv;
                            }
                    }
                    // explicit reflector: 0 above j, 1 at j, v below, 0 past rb (x is 0 there)
                    T* vj = S.Vp + jj * ldvp;
                    const T vmine = lane > jl ? xs : (lane == jl ? T(1) : T(0));
                    vj[rh] = vmine;
                    T* vt = vj + tb + lane;
#pragma unroll
                    for (int t4 = 0; t4 < kGRPL / 4; ++t4)
                        if (t4 < nt4) {
                            vt[128 * t4] = x[4 * t4];
                            vt[128 * t4 + 32] = x[4 * t4 + 1];
                            vt[128 * t4 + 64] = x[4 * t4 + 2];
                            vt[128 * t4 + 96] = x[4 * t4 + 3];
                        }
                    if (lane == 0) S.beta[j] = bj;
                    if (jj + 1 < nbp) named_bar_arrive(bar, cnt);
                    // Off the chain: G(a, w) = v_a^T v_w for the earlier reflectors of the panel (the
                    // compact-WY recurrence needs the strict upper triangle), from the registers that
                    // still hold v_w — instead of a 16 x 16 x K CTA GEMM after the panel.
                    for (int a = 0; a < jj; ++a) {
                        const T* va = S.Vp + a * ldvp + tb + lane;
                        T g0 = S.Vp[a * ldvp + rh] * vmine, g1 = 0, g2 = 0, g3 = 0;
#pragma unroll
                        for (int t4 = 0; t4 < kGRPL / 4; ++t4)
                            if (t4 < nt4) {
                                g0 += va[128 * t4] * x[4 * t4];
                                g1 += va[128 * t4 + 32] * x[4 * t4 + 1];
                                g2 += va[128 * t4 + 64] * x[4 * t4 + 2];
                                g3 += va[128 * t4 + 96] * x[4 * t4 + 3];
                            }
                        const T gsum = warp_sum((g0 + g1) + (g2 + g3));
                        if (lane == 0) S.Gp[a * kNB + jj] = gsum;
                    }
                }
            }
            if (rh >= p0 && rh < rb) col[rh] = xs;
#pragma unroll
            for (int t4 = 0; t4 < kGRPL / 4; ++t4)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int r = tb + 32 * (4 * t4 + q4) + lane;
                    if (t4 < nt4 && r < rb) col[r] = x[4 * t4 + q4];
                }
        } else if (warp < nbp) {
            const int c = p0 + warp;
            T* col = W + int64_t(c) * ldv;
            for (int jj = 0; jj <= warp; ++jj) {
                const int j = p0 + jj;
                const int bar = 1 + jj, cnt = 32 * (nbp - jj);
                if (jj < warp) {
                    named_bar_sync(bar, cnt);
                    const T bj = S.beta[j];
                    if (bj == T(0)) continue;
                    const T* vj = S.Vp + jj * ldvp;
                    T s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                    int i = j + lane;
                    for (; i + 96 < rb; i += 128) {
                        s0 += vj[i] * col[i];
                        s1 += vj[i + 32] * col[i + 32];
                        s2 += vj[i + 64] * col[i + 64];
                        s3 += vj[i + 96] * col[i + 96];
                    }
                    for (; i < rb; i += 32) s0 += vj[i] * col[i];
                    const T s = warp_sum((s0 + s1) + (s2 + s3)) * bj;
                    for (int i2 = j + lane; i2 < rb; i2 += 32) col[i2] -= s * vj[i2];
                    __syncwarp();
                } else {
                    T q0 = 0, q1 = 0;
                    int i = j + 1 + lane;
                    for (; i + 32 < rb; i += 64) {
                        q0 += col[i] * col[i];
                        q1 += col[i + 32] * col[i + 32];
                    }
                    for (; i < rb; i += 32) q0 += col[i] * col[i];
                    const T sig = warp_sum(q0 + q1);
                    const T x0 = col[j];
                    T bj = 0;
                    if (sig != T(0)) {
                        T mu, v0, rv;
                        reflector_scalars(x0, sig, mu, v0, bj, rv);
                        for (int i2 = j + 1 + lane; i2 < rb; i2 += 32) col[i2] *= rv;
                        __syncwarp();
                        if (lane == 0) col[j] = mu;
                    }
                    __syncwarp();
                    T* vj = S.Vp + jj * ldvp;
                    for (int i2 = lane; i2 < ldvp; i2 += 32)
                        vj[i2] = (i2 > j && i2 < rb) ? col[i2] : T(i2 == j ? 1 : 0);
                    if (lane == 0) S.beta[j] = bj;
                    __threadfence_block();
                    if (jj + 1 < nbp) named_bar_arrive(bar, cnt);
                }
            }
        }
        __syncthreads();
        QRG_ADD(1, tq);
        const int K = rb - p0;
        if (!reg_panel) {
            cta_mm(nbp, nbp, K, S.Vp + p0, ldvp, 1, S.Vp + p0, 1, ldvp, S.Gp, kNB, 1, T(1), false, S.scratch, kGemmScratch);
            __syncthreads();
        }
        QRG_ADD(2, tq);
        if (warp == 0) {
            warp_larft<T>(nbp, S.Gp, kNB, S.beta + p0, S.Tp, kNB);
            T* Tpg = Tb + pi * kNB * kNB;
            for (int e = lane; e < kNB * kNB; e += 32) Tpg[e] = S.Tp[e];
        }
        __syncthreads();
        QRG_ADD(3, tq);
        const int c0 = p0 + nbp, nc = d - c0;
        if (nc > 0) {
            T* C = W + int64_t(c0) * ldv + p0;
            cta_mm(nbp, nc, K, S.Vp + p0, ldvp, 1, C, 1, ldv, S.Y, d, 1, T(1), false, S.scratch, kGemmScratch);
            __syncthreads();
            QRG_ADD(4, tq);
            cta_mm(nbp, nc, nbp, S.Tp, 1, kNB, S.Y, d, 1, S.Z, d, 1, T(1), false, S.scratch, kGemmScratch);
            __syncthreads();
            QRG_ADD(5, tq);
            if constexpr (sizeof(T) == 8)
                cta_rank_update_global(K, nc, nbp, reinterpret_cast<const double*>(S.Vp + p0), ldvp,
                                       reinterpret_cast<const double*>(S.Z), d, reinterpret_cast<double*>(C), ldv);
            else
                cta_mm(K, nc, nbp, S.Vp + p0, 1, ldvp, S.Z, d, 1, C, 1, ldv, T(-1), true, S.scratch, kGemmScratch);
            __syncthreads();
            QRG_ADD(6, tq);
        }
    }
    for (int e = tid; e < d * d; e += kBThreads) {
        const int r = e / d, c = e % d;
        Rout[(int64_t(b) * d + r) * ldr + c] = (r <= c) ? W[int64_t(c) * ldv + r] : T(0);
    }
    for (int c = tid; c < d; c += kBThreads) betas[int64_t(b) * d + c] = S.beta[c];
    __syncthreads();
    for (int c = warp; c < d; c += kBThreads / 32)  // explicit reflectors in place
        for (int r = lane; r <= c && r < rb; r += 32) W[int64_t(c) * ldv + r] = T(r == c ? 1 : 0);
    QRG_ADD(7, tq);
}

template <typename T>
struct FormQSmem {
    int ldvs, lde;
    T *Vs, *E, *Y, *Z, *Tp, *scratch;
    // stage: 0 = reflectors read from global, 1 = all d reflector columns staged in shared memory;
    // qc = Q columns formed by this CTA
    __device__ FormQSmem(unsigned char* raw, int d, int rb, int stage, int qc) : ldvs(ld_mod(rb, 8)), lde(ld_mod(rb, 4)) {
        T* p = reinterpret_cast<T*>(raw);
        E = p;
        p += size_t(qc) * lde;
        Y = p;
        p += kNB * qc;
        Z = p;
        p += kNB * qc;
        Tp = p;
        p += kNB * kNB;
        scratch = p;
        p += kGemmScratch;
        Vs = stage ? p : nullptr;
    }
    static size_t bytes(int d, int rb, size_t eb, int stage, int qc) {
        return (size_t(qc) * ld_mod(rb, 4) + 2 * kNB * qc + kNB * kNB + kGemmScratch +
                (stage == 1 ? size_t(d) * ld_mod(rb, 8) : 0)) *
               eb;
    }
};
// Staging mode of a level: all reflector columns staged when they fit next to the 32-column chunk
// (small blocks); big blocks read them from L2. (Staging one panel at a time with 16-column chunks
// was measured slower at C3: 7 chunk CTAs per block instead of 4, 5.0 vs 4.0 ms for the tree.)
template <typename T>
inline void formq_mode(int d, int rb, int max_smem, int* stage, int* qc) {
    *qc = kQChunk;
    *stage = FormQSmem<T>::bytes(d, rb, sizeof(T), 1, kQChunk) <= size_t(max_smem) ? 1 : 0;
}

// Q block b = H_0 ... H_{d-1} [Qin_b; 0]  (Qin null => identity), by panels in reverse:
//   E <- E - V_p (T_p (V_p^T E)),  p = P-1 ... 0. Columns of Q are independent, so each CTA
//   forms one qc-wide column chunk (grid = blocks x chunks) to spread a level over more SMs.
//   V is the explicit reflector matrix (column-major, ldv), staged in shared memory when it fits.
template <typename T>
__global__ void __launch_bounds__(kBThreads, 1)
    k_qr_blocked_form_q(const T* __restrict__ Qin, int ldqin, int64_t rows, int nb, int d, const T* __restrict__ V,
                        int ldv, const T* __restrict__ Tg, T* __restrict__ Qout, int64_t ldqout, int stage, int qc,
                        const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    FormQSmem<T> S(smem_raw, d, rb, stage, qc);
    const T* Vb = V + int64_t(b) * d * ldv;
    const T* Tb = Tg + int64_t(b) * npanels(d) * kNB * kNB;
    const T* Qb = Qin ? Qin + int64_t(b) * d * ldqin : nullptr;
    const T* Vx = Vb;
    int ldx = ldv;
    if (stage == 1) {
        for (int c = warp; c < d; c += kBThreads / 32)
            for (int r = lane; r < rb; r += 32) S.Vs[c * S.ldvs + r] = Vb[int64_t(c) * ldv + r];
        Vx = S.Vs;
        ldx = S.ldvs;
    }
    const int q0 = blockIdx.y * qc;  // this CTA's column chunk of Q
    const int nq = min(qc, d - q0);
    for (int j = warp; j < nq; j += kBThreads / 32)
        for (int i = lane; i < rb; i += 32)
            S.E[j * S.lde + i] = i < d ? (Qb ? Qb[i * ldqin + q0 + j] : T(i == q0 + j ? 1 : 0)) : T(0);
    __syncthreads();
    for (int pi = npanels(d) - 1; pi >= 0; --pi) {
        const int p0 = pi * kNB, nbp = min(kNB, d - p0), K = rb - p0;
        const T* Vp = Vx + p0 * ldx + p0;  // V_p rows >= p0
        const int ldp = ldx;
        if (tid < kNB * kNB) S.Tp[tid] = Tb[pi * kNB * kNB + tid];
        if constexpr (std::is_same<T, double>::value) {
            if (stage == 0 && nq <= 32)
                cta_vt_e_ga(nbp, nq, K, Vp, ldp, S.E + p0, S.lde, S.Y, qc, S.scratch, kGemmScratch);
            else
                cta_mm(nbp, nq, K, Vp, ldp, 1, S.E + p0, 1, S.lde, S.Y, qc, 1, T(1), false, S.scratch, kGemmScratch);
        } else {
            cta_mm(nbp, nq, K, Vp, ldp, 1, S.E + p0, 1, S.lde, S.Y, qc, 1, T(1), false, S.scratch, kGemmScratch);
        }
        __syncthreads();
        cta_mm(nbp, nq, nbp, S.Tp, kNB, 1, S.Y, qc, 1, S.Z, qc, 1, T(1), false, S.scratch, kGemmScratch);
        __syncthreads();
        if constexpr (std::is_same<T, double>::value) {
            if (stage == 0 && nq <= 32)  // reflectors in L2: the strip kernel (same bits, ~9x fewer instructions)
                cta_strip_update_ga(K, nq, nbp, Vp, ldp, S.Z, qc, S.E + p0, S.lde);
            else
                cta_mm(K, nq, nbp, Vp, 1, ldp, S.Z, qc, 1, S.E + p0, 1, S.lde, T(-1), true, S.scratch, kGemmScratch);
        } else {
            cta_mm(K, nq, nbp, Vp, 1, ldp, S.Z, qc, 1, S.E + p0, 1, S.lde, T(-1), true, S.scratch, kGemmScratch);
        }
        __syncthreads();
    }
    T* Qo = Qout + r0 * ldqout + q0;
    if (nq == 32) {
        for (int e = tid; e < 32 * rb; e += kBThreads) {
            const int i = e >> 5, j = e & 31;
            Qo[int64_t(i) * ldqout + j] = S.E[j * S.lde + i];
        }
    } else {
        for (int e = tid; e < nq * rb; e += kBThreads) {
            const int i = e / nq, j = e % nq;
            Qo[int64_t(i) * ldqout + j] = S.E[j * S.lde + i];
        }
    }
}

// ============================================================================================
// Register-resident path for narrow sketches (d <= 64, blocks of <= 256 rows: C1, C2). The d
// reflector steps are the latency chain, so the factor kernel keeps the whole block in registers
// (warp w owns columns w, w+16, ...; lane l holds rows l, l+32, ...) and runs ONE block barrier
// per column: after applying H_j to its trailing columns (apply_reflector, qr.hpp:49-57), the warp
// that owns column j+1 immediately builds reflector j+1 (make_reflector, qr.hpp:32-45) into a
// double-buffered shared slot; after the barrier every warp applies it. The Q kernel keeps
// [Q_above; 0] in registers the same way and applies the stored reflectors backwards
// (accumulate_q order, qr.hpp:60-72) without any barrier. Scalar formulas use uncontracted
// _rn operations like the reference; the reductions are tree-ordered.
constexpr int kRegWarps = 16;
constexpr int kRegRPL = 8;  // rows per lane: blocks of <= 256 rows

template <typename T> __device__ __forceinline__ T mul_rn_t(T a, T b);
template <> __device__ __forceinline__ double mul_rn_t<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn_t<float>(float a, float b) { return __fmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn_t(T a, T b);
template <> __device__ __forceinline__ double add_rn_t<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float add_rn_t<float>(float a, float b) { return __fadd_rn(a, b); }

template <typename T, int CPW>
__global__ void __launch_bounds__(kRegWarps * 32, 1)
    k_qr_reg(const T* __restrict__ X, int64_t ldx, int64_t rows, int nb, int d, T* __restrict__ V, int ldv,
             T* __restrict__ betas, T* __restrict__ Rout, int ldr, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    constexpr int RPL = kRegRPL, R = RPL * 32, NW = kRegWarps;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* slot_v = reinterpret_cast<T*>(smem_raw);  // [2][R]
    T* slot_b = slot_v + 2 * R;                  // [2]
    T* W = slot_b + 2;                           // staging, column-major [d][R + 1]
    constexpr int ldw = R + 1;
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // coalesced row-major load -> column-major staging -> registers
    for (int e = tid; e < rb * d; e += NW * 32) {
        const int r = e / d, c = e % d;
        W[c * ldw + r] = X[(r0 + r) * ldx + c];
    }
    __syncthreads();
    T col[CPW][RPL];
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const int c = warp + NW * k;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
            const int r = lane + 32 * u;
            col[k][u] = (c < d && r < rb) ? W[c * ldw + r] : T(0);
        }
    }
    // make_reflector for column jn (owned by this warp as col[kk]); publishes into slot sl.
    auto build = [&](int jn, int kk, int sl) {
        T x[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
            x[u] = col[0][u];
#pragma unroll
            for (int k = 1; k < CPW; ++k) x[u] = (k == kk) ? col[k][u] : x[u];
        }
        T sig = 0, x0 = 0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
            const int r = lane + 32 * u;
            if (r > jn) sig = add_rn_t(sig, mul_rn_t(x[u], x[u]));
            if (r == jn) x0 = x[u];
        }
        sig = warp_sum(sig);
        x0 = __shfl_sync(0xffffffffu, x0, jn & 31);
        T* v = slot_v + sl * R;
        T beta = 0;
        if (sig != T(0)) {
            T mu, v0, rv;
            reflector_scalars(x0, sig, mu, v0, beta, rv);
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int r = lane + 32 * u;
                v[r] = r > jn && r < rb ? mul_rn_t(x[u], rv) : T(r == jn ? 1 : 0);
                if (r == jn) {
#pragma unroll
                    for (int k = 0; k < CPW; ++k)
                        if (k == kk) col[k][u] = mu;  // R(jn, jn) = mu
                }
            }
        } else {  // sigma == 0: no reflection, the diagonal keeps its value (qr.hpp:37)
#pragma unroll
            for (int u = 0; u < RPL; ++u) v[lane + 32 * u] = T(0);
        }
        if (lane == 0) slot_b[sl] = beta;
    };
    if (warp == 0) build(0, 0, 0);
    __syncthreads();
    T* Vb = V + int64_t(b) * d * ldv;
    for (int j = 0; j < d; ++j) {
        const int sl = j & 1;
        QRR_CLK(t0, 0);
        const T beta = slot_b[sl];
        T v[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) v[u] = slot_v[sl * R + lane + 32 * u];
        QRR_CLK(t1, v[RPL - 1] + beta);
        if (warp == j % NW) {  // the owner of column j stores reflector j for the Q kernel
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int r = lane + 32 * u;
                if (r < ldv) Vb[int64_t(j) * ldv + r] = r < rb ? v[u] : T(0);
            }
            if (lane == 0) betas[int64_t(b) * d + j] = beta;
        }
        if (beta != T(0)) {
            T sk[CPW];
#pragma unroll
            for (int k = 0; k < CPW; ++k) {
                sk[k] = 0;
#pragma unroll
                for (int u = 0; u < RPL; ++u) sk[k] += v[u] * col[k][u];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int k = 0; k < CPW; ++k) sk[k] += __shfl_xor_sync(0xffffffffu, sk[k], o);
#pragma unroll
            for (int k = 0; k < CPW; ++k) {
                const int c = warp + NW * k;
                if (c > j && c < d) {
                    const T sb = sk[k] * beta;
#pragma unroll
                    for (int u = 0; u < RPL; ++u) col[k][u] = add_rn_t(col[k][u], -mul_rn_t(sb, v[u]));
                }
            }
        }
        QRR_CLK(t2, col[CPW - 1][RPL - 1]);
        if (j + 1 < d && warp == (j + 1) % NW) build(j + 1, (j + 1) / NW, sl ^ 1);
        QRR_CLK(t3, col[0][0]);
        __syncthreads();
        QRR_CLK(t4, 0);
        if (warp == 0) { QRR_ADD(0, t1 - t0); QRR_ADD(1, t2 - t1); QRR_ADD(2, t3 - t2); QRR_ADD(3, t4 - t3); }
        if (j + 1 < d && warp == (j + 1) % NW) { QRR_ADD(4, t1 - t0); QRR_ADD(5, t2 - t1); QRR_ADD(6, t3 - t2); QRR_ADD(7, t4 - t3); }
    }
    // R (upper triangle, exact zeros below; qr.hpp:74-79) -> rows [b*d, (b+1)*d) of Rout
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const int c = warp + NW * k;
        if (c < d) {
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int r = lane + 32 * u;
                if (r < d) Rout[(int64_t(b) * d + r) * ldr + c] = r <= c ? col[k][u] : T(0);
            }
        }
    }
}

// Q block b = H_0 ... H_{d-1} [Qin_b; 0] (Qin null => identity), rows [r0, r1) of Qout.
template <typename T, int CPW>
__global__ void __launch_bounds__(kRegWarps * 32, 1)
    k_qr_reg_form_q(const T* __restrict__ Qin, int ldqin, int64_t rows, int nb, int d, const T* __restrict__ V,
                    int ldv, const T* __restrict__ betas, T* __restrict__ Qout, int64_t ldqout, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // CholeskyQR2 already produced this QR (cholqr.cu)
    constexpr int RPL = kRegRPL, R = RPL * 32, NW = kRegWarps;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Vs = reinterpret_cast<T*>(smem_raw);  // [d][R] reflectors, later the output staging [d][R+1]
    T* sb = Vs + size_t(d) * (R + 1);        // [d] betas
    const int b = blockIdx.x;
    const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
    const int rb = int(r1 - r0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T* Vb = V + int64_t(b) * d * ldv;
    for (int e = tid; e < d * R; e += NW * 32) {
        const int c = e / R, r = e % R;
        Vs[c * R + r] = r < rb ? Vb[int64_t(c) * ldv + r] : T(0);
    }
    for (int c = tid; c < d; c += NW * 32) sb[c] = betas[int64_t(b) * d + c];
    T col[CPW][RPL];
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const int c = warp + NW * k;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
            const int r = lane + 32 * u;
            T x = T(0);
            if (c < d && r < d) x = Qin ? Qin[(int64_t(b) * d + r) * ldqin + c] : T(r == c ? 1 : 0);
            col[k][u] = x;
        }
    }
    __syncthreads();
    for (int j = d - 1; j >= 0; --j) {
        const T beta = sb[j];
        if (beta == T(0)) continue;
        T v[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) v[u] = Vs[j * R + lane + 32 * u];
        T sk[CPW];
#pragma unroll
        for (int k = 0; k < CPW; ++k) {
            sk[k] = 0;
#pragma unroll
            for (int u = 0; u < RPL; ++u) sk[k] += v[u] * col[k][u];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int k = 0; k < CPW; ++k) sk[k] += __shfl_xor_sync(0xffffffffu, sk[k], o);
#pragma unroll
        for (int k = 0; k < CPW; ++k) {
            const T s2 = sk[k] * beta;
#pragma unroll
            for (int u = 0; u < RPL; ++u) col[k][u] = add_rn_t(col[k][u], -mul_rn_t(s2, v[u]));
        }
    }
    __syncthreads();  // reuse Vs as the output staging
    constexpr int ldo = R + 1;
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const int c = warp + NW * k;
        if (c < d) {
#pragma unroll
            for (int u = 0; u < RPL; ++u) Vs[c * ldo + lane + 32 * u] = col[k][u];
        }
    }
    __syncthreads();
    for (int e = tid; e < rb * d; e += NW * 32) {
        const int r = e / d, c = e % d;
        Qout[(r0 + r) * ldqout + c] = Vs[c * ldo + r];
    }
}

size_t reg_factor_smem_bytes(int d, size_t eb) { return (2 * size_t(kRegRPL * 32) + 2 + size_t(d) * (kRegRPL * 32 + 1)) * eb; }
size_t reg_formq_smem_bytes(int d, size_t eb) { return (size_t(d) * (kRegRPL * 32 + 1) + d) * eb; }

size_t wide_factor_smem_bytes(int rbmax, int d, size_t eb) {
    return ((d * 4 + 15) / 16) * 16 + ((d + 1) / 2) * 2 * eb + size_t(rbmax | 1) * d * eb;
}


}  // namespace

TsqrPlan plan_tsqr(int64_t m, int d, size_t eb, int max_smem, int num_sms) {
    TsqrPlan p;
    p.m = m;
    p.d = d;
    p.elem_bytes = eb;
    const size_t cap = size_t(max_smem);
    // Largest block for the shared-memory blocked kernels (<= 256 rows, register panels).
    int rb_blocked = 0;
    for (int rb = kMaxRowsBlocked; rb > d; --rb)
        if (BlockedSmem<double>::bytes(d, rb, eb) <= cap && FormQSmem<double>::bytes(d, rb, eb, 1, kQChunk) <= cap) {
            rb_blocked = rb;
            break;
        }
    // Largest block for the global-working-set blocked kernels (panel reflectors + Q chunk in smem).
    int rb_big = 0;
    for (int rb = 4096; rb > d; --rb)
        if (BigSmem<double>::bytes(d, rb, eb) <= cap && FormQSmem<double>::bytes(d, rb, eb, 0, kQChunk) <= cap) {
            rb_big = rb;
            break;
        }
    const bool big_ok = rb_big >= 2 * d + 2;
    // Narrow sketches: the register-resident kernels (one barrier per column) on <= 256-row blocks.
#ifdef CORU_TSQR_REG  // tooling: the register-resident kernels (slower than the blocked ones on B200)
    const bool reg_ok = d <= 64 && reg_factor_smem_bytes(d, eb) <= cap && reg_formq_smem_bytes(d, eb) <= cap;
#else
    const bool reg_ok = false;
#endif
    // The shared-memory kernels are fastest per block, but when they cannot reduce a level by at
    // least 2x (wide sketches: d = 110 fits only ~168 rows) the tree gets deep and every level
    // costs d sequential reflector steps; then the L2-resident kernels with ~1024-row blocks win.
    const bool blocked_ok = rb_blocked >= 2 * d + 2 || (rb_blocked >= d + 1 + d / 4 && !big_ok);
    int target;
    if (reg_ok) target = kRegRPL * 32;
    else if (blocked_ok) target = rb_blocked;
    else if (big_ok) target = std::min(rb_big, std::max(4 * d, 1024));
    else target = std::max(4 * d, 256);
    if (const char* e = getenv("CORU_TSQR_TARGET")) target = std::max(atoi(e), d + 1);  // tooling: tree shape sweeps
    int64_t rows = m;
    int64_t voff = 0, boff = 0, roff = 0, toff = 0;
    for (;;) {
        TsqrLevel L;
        L.rows = rows;
        // every block strictly taller than d (so the tree always shrinks), at most `target` rows
        int64_t nb = std::max<int64_t>(1, (rows + target - 1) / target);
        // one CTA per block and SM: a level of more blocks than SMs runs in whole waves, so round
        // the block count up to a multiple of the SM count (C3 level 0: 249 blocks of 803 rows were
        // two waves; 296 blocks of 676 rows are two FULL waves of shorter blocks)
        if (nb > num_sms) nb = (nb + num_sms - 1) / num_sms * num_sms;
        nb = std::max<int64_t>(1, std::min<int64_t>(nb, rows / (d + 1)));
        L.nb = int(nb);
        L.rbmax = int((rows + nb - 1) / nb);
        if (reg_ok && L.rbmax <= kRegRPL * 32) {
            L.kind = TsqrLevel::kReg;
        } else if (blocked_ok && L.rbmax <= rb_blocked) {
            L.kind = TsqrLevel::kBlockedSmem;
        } else if (rb_big > d && L.rbmax <= rb_big) {
            L.kind = TsqrLevel::kBlockedGlobal;
        } else {
            L.kind = TsqrLevel::kWide;
        }
        L.blocked = L.kind == TsqrLevel::kBlockedSmem || L.kind == TsqrLevel::kBlockedGlobal;
        L.smem = L.kind == TsqrLevel::kBlockedSmem || L.kind == TsqrLevel::kReg ||
                 (L.kind == TsqrLevel::kWide && wide_factor_smem_bytes(L.rbmax, d, eb) <= cap);
        L.ldv = L.rbmax + (L.rbmax % 2);
        L.v_off = voff;
        L.beta_off = boff;
        L.r_off = roff;
        L.t_off = toff;
        voff += int64_t(L.nb) * d * L.ldv;
        boff += int64_t(L.nb) * d;
        roff += int64_t(L.nb) * d * d;
        if (L.blocked) toff += int64_t(L.nb) * npanels(d) * kNB * kNB;
        p.levels.push_back(L);
        if (L.nb == 1) break;
        rows = int64_t(L.nb) * d;  // < previous rows: each block has > d rows
    }
    p.blocked = !p.levels.empty() && p.levels[0].blocked;
    p.v_elems = voff;
    p.beta_elems = boff;
    p.r_elems = roff;
    p.t_elems = toff;
    p.max_smem = max_smem;
    return p;
}

int64_t tsqr_scratch_elems(const TsqrPlan& p) {
    int64_t work = 0, maxrows = 0;
    for (size_t l = 0; l < p.levels.size(); ++l) {
        const TsqrLevel& L = p.levels[l];
        if (!L.blocked && !L.smem) work = std::max<int64_t>(work, int64_t(L.nb) * p.d * L.ldv);
        if (l >= 1) maxrows = std::max<int64_t>(maxrows, L.rows);
    }
    return work + 2 * maxrows * p.d;
}

template <typename T>
cudaError_t tsqr_factor(const TsqrPlan& p, const T* B, int64_t ldb, T* V, T* beta, T* Tarena, T* R, T* r_out,
                        cudaStream_t st, const int* gate) {
    const int d = p.d;
    const T* X = B;
    int64_t ldx = ldb;
    for (size_t l = 0; l < p.levels.size(); ++l) {
        const TsqrLevel& L = p.levels[l];
        T* Rl = (l + 1 == p.levels.size()) ? r_out : R + L.r_off;
        if (L.kind == TsqrLevel::kReg) {
            const size_t sm = reg_factor_smem_bytes(d, sizeof(T));
            if (d <= 32) {
                allow_max_smem(k_qr_reg<T, 2>);
                k_qr_reg<T, 2><<<L.nb, kRegWarps * 32, sm, st>>>(X, ldx, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                                 beta + L.beta_off, Rl, d, gate);
            } else {
                allow_max_smem(k_qr_reg<T, 4>);
                k_qr_reg<T, 4><<<L.nb, kRegWarps * 32, sm, st>>>(X, ldx, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                                 beta + L.beta_off, Rl, d, gate);
            }
        } else if (L.kind == TsqrLevel::kBlockedSmem) {
            const size_t sm = BlockedSmem<T>::bytes(d, L.rbmax, sizeof(T));
            allow_max_smem(k_qr_blocked<T>);
            k_qr_blocked<T><<<L.nb, kBThreads, sm, st>>>(X, ldx, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                          beta + L.beta_off, Tarena + L.t_off, Rl, d, gate);
        } else if (L.kind == TsqrLevel::kBlockedGlobal) {
            const size_t sm = BigSmem<T>::bytes(d, L.rbmax, sizeof(T));
            allow_max_smem(k_qr_blocked_g<T>);
            k_qr_blocked_g<T><<<L.nb, kBThreads, sm, st>>>(X, ldx, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                            beta + L.beta_off, Tarena + L.t_off, Rl, d, gate);
        } else {
            const size_t sm = L.smem ? wide_factor_smem_bytes(L.rbmax, d, sizeof(T)) : wide_factor_smem_bytes(0, d, sizeof(T));
            allow_max_smem(k_hh_factor<T>);
            k_hh_factor<T><<<L.nb, kThreads, sm, st>>>(X, ldx, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                        beta + L.beta_off, Rl, d, L.smem ? 1 : 0, gate);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        X = Rl;
        ldx = d;
    }
    return cudaSuccess;
}

template <typename T>
cudaError_t tsqr_form_q(const TsqrPlan& p, const T* q_top, T* V, T* beta, T* Tarena, T* scratch, T* Q, int64_t ldq,
                        int max_smem, cudaStream_t st, const int* gate) {
    const int d = p.d;
    // scratch = [wide-path working blocks | ping | pong]
    int64_t work = 0, maxrows = 0;
    for (size_t l = 0; l < p.levels.size(); ++l) {
        const TsqrLevel& L = p.levels[l];
        if (!L.blocked && !L.smem) work = std::max<int64_t>(work, int64_t(L.nb) * d * L.ldv);
        if (l >= 1) maxrows = std::max<int64_t>(maxrows, L.rows);
    }
    T* ping = scratch + work;
    T* pong = ping + maxrows * d;
    const T* qin = q_top;
    int ldqin = d;
    for (int l = int(p.levels.size()) - 1; l >= 0; --l) {
        const TsqrLevel& L = p.levels[size_t(l)];
        T* out = (l == 0) ? Q : ((p.levels.size() - 1 - size_t(l)) % 2 == 0 ? ping : pong);
        const int64_t ldo = (l == 0) ? ldq : d;
        if (L.kind == TsqrLevel::kReg) {
            const size_t sm = reg_formq_smem_bytes(d, sizeof(T));
            if (d <= 32) {
                allow_max_smem(k_qr_reg_form_q<T, 2>);
                k_qr_reg_form_q<T, 2><<<L.nb, kRegWarps * 32, sm, st>>>(qin, ldqin, L.rows, L.nb, d, V + L.v_off,
                                                                        L.ldv, beta + L.beta_off, out, ldo, gate);
            } else {
                allow_max_smem(k_qr_reg_form_q<T, 4>);
                k_qr_reg_form_q<T, 4><<<L.nb, kRegWarps * 32, sm, st>>>(qin, ldqin, L.rows, L.nb, d, V + L.v_off,
                                                                        L.ldv, beta + L.beta_off, out, ldo, gate);
            }
        } else if (L.blocked) {
            int stage = 0, qc = kQChunk;
            formq_mode<T>(d, L.rbmax, max_smem, &stage, &qc);
            const size_t sm = FormQSmem<T>::bytes(d, L.rbmax, sizeof(T), stage, qc);
            allow_max_smem(k_qr_blocked_form_q<T>);
            const dim3 grid(unsigned(L.nb), unsigned((d + qc - 1) / qc));
            k_qr_blocked_form_q<T><<<grid, kBThreads, sm, st>>>(qin, ldqin, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                                 Tarena + L.t_off, out, ldo, stage, qc, gate);
        } else {
            const size_t sm = L.smem ? size_t(L.rbmax | 1) * d * sizeof(T) : 0;
            allow_max_smem(k_hh_form_q<T>);
            k_hh_form_q<T><<<L.nb, kThreads, sm, st>>>(qin, ldqin, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                        beta + L.beta_off, out, ldo, scratch, L.smem ? 1 : 0, gate);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        qin = out;
        ldqin = int(ldo);
    }
    return cudaSuccess;
}

template cudaError_t tsqr_factor<double>(const TsqrPlan&, const double*, int64_t, double*, double*, double*, double*,
                                         double*, cudaStream_t, const int*);
template cudaError_t tsqr_factor<float>(const TsqrPlan&, const float*, int64_t, float*, float*, float*, float*, float*,
                                        cudaStream_t, const int*);
template cudaError_t tsqr_form_q<double>(const TsqrPlan&, const double*, double*, double*, double*, double*, double*,
                                         int64_t, int, cudaStream_t, const int*);
template cudaError_t tsqr_form_q<float>(const TsqrPlan&, const float*, float*, float*, float*, float*, float*, int64_t,
                                        int, cudaStream_t, const int*);

}  // namespace coru_gpu

#ifdef CORU_QR_PROFILE
// Tooling (tools/qrg_phases.py, a -DCORU_QR_PROFILE build): cycles block 0 of k_qr_blocked_g spent
// per phase since the last reset.
extern "C" int coru_debug_qrg_phases(long long* out, int reset) {
    long long z[12] = {};
    if (cudaMemcpyFromSymbol(out, coru_gpu::g_qrg_phase, sizeof(z)) != cudaSuccess) return 1;
    if (reset && cudaMemcpyToSymbol(coru_gpu::g_qrg_phase, z, sizeof(z)) != cudaSuccess) return 1;
    return 0;
}
#endif
