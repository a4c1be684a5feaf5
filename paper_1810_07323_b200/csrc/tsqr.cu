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
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "tsqr.cuh"

namespace coru_gpu {

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
    const T mu = tsqrt(x0 * x0 + sig);
    const T v0 = (x0 <= T(0)) ? x0 - mu : -sig / (x0 + mu);
    const T beta = T(2) * v0 * v0 / (sig + v0 * v0);
    for (int i = j + 1 + lane; i < rb; i += 32) col[i] /= v0;
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
                                                        T* __restrict__ Rout, int ldr, int use_smem) {
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
                                                        int64_t ldqout, T* __restrict__ gscratch, int use_smem) {
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

size_t factor_smem_bytes(int rbmax, int d, size_t eb) {
    return ((d * 4 + 15) / 16) * 16 + ((d + 1) / 2) * 2 * eb + size_t(rbmax | 1) * d * eb;
}

}  // namespace

TsqrPlan plan_tsqr(int64_t m, int d, size_t eb, int max_smem) {
    TsqrPlan p;
    p.m = m;
    p.d = d;
    p.elem_bytes = eb;
    // Largest block that fits shared memory; prefer ~4d..512 rows per block.
    int rb_smem = 0;
    for (int rb = 2048; rb > d; rb -= 1)
        if (factor_smem_bytes(rb, d, eb) <= size_t(max_smem)) { rb_smem = rb; break; }
    const bool smem = rb_smem >= 2 * d + 2;
    int target = smem ? std::min(rb_smem, std::max(4 * d, 256)) : std::max(4 * d, 256);
    int64_t rows = m;
    int64_t voff = 0, boff = 0, roff = 0;
    for (;;) {
        TsqrLevel L;
        L.rows = rows;
        L.smem = smem;
        int64_t nb = (rows + target - 1) / target;
        nb = std::min<int64_t>(nb, rows / (d + 1));  // every block strictly taller than d
        if (nb < 1) nb = 1;
        L.nb = int(nb);
        L.rbmax = int((rows + nb - 1) / nb);
        if (L.smem && factor_smem_bytes(L.rbmax, d, eb) > size_t(max_smem)) L.smem = false;
        L.ldv = L.rbmax + (L.rbmax % 2);
        L.v_off = voff;
        L.beta_off = boff;
        L.r_off = roff;
        voff += int64_t(L.nb) * d * L.ldv;
        boff += int64_t(L.nb) * d;
        roff += int64_t(L.nb) * d * d;
        p.levels.push_back(L);
        if (L.nb == 1) break;
        rows = int64_t(L.nb) * d;
    }
    p.v_elems = voff;
    p.beta_elems = boff;
    p.r_elems = roff;
    return p;
}

int64_t tsqr_scratch_elems(const TsqrPlan& p) {
    int64_t s = 0;
    for (auto& L : p.levels)
        if (!L.smem) s = std::max<int64_t>(s, int64_t(L.nb) * p.d * L.ldv);
    return s;
}

template <typename T>
cudaError_t tsqr_factor(const TsqrPlan& p, const T* B, int64_t ldb, T* V, T* beta, T* R, T* r_out,
                        cudaStream_t st) {
    const int d = p.d;
    const T* X = B;
    int64_t ldx = ldb;
    for (size_t l = 0; l < p.levels.size(); ++l) {
        const TsqrLevel& L = p.levels[l];
        const size_t sm = L.smem ? factor_smem_bytes(L.rbmax, d, sizeof(T)) : factor_smem_bytes(0, d, sizeof(T));
        cudaFuncSetAttribute(k_hh_factor<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        T* Rl = (l + 1 == p.levels.size()) ? r_out : R + L.r_off;
        k_hh_factor<T><<<L.nb, kThreads, sm, st>>>(X, ldx, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                    beta + L.beta_off, Rl, d, L.smem ? 1 : 0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        X = Rl;
        ldx = d;
    }
    return cudaSuccess;
}

template <typename T>
cudaError_t tsqr_form_q(const TsqrPlan& p, const T* q_top, T* V, T* beta, T* scratch, T* Q, int64_t ldq,
                        cudaStream_t st) {
    const int d = p.d;
    // Level l's output Q (rows_l x d) is the Qin of level l-1. Intermediate Qs go to scratch
    // space carved from the R arena region sizes: reuse a ping-pong pair in `scratch` tail.
    // Layout: scratch holds [global-L2 working blocks | ping | pong].
    const int64_t work = tsqr_scratch_elems(p);
    int64_t maxrows = 0;
    for (size_t l = 1; l < p.levels.size(); ++l) maxrows = std::max<int64_t>(maxrows, p.levels[l].rows);
    T* ping = scratch + work;
    T* pong = ping + maxrows * d;
    const T* qin = q_top;
    int ldqin = d;
    for (int l = int(p.levels.size()) - 1; l >= 0; --l) {
        const TsqrLevel& L = p.levels[size_t(l)];
        T* out = (l == 0) ? Q : ((p.levels.size() - 1 - size_t(l)) % 2 == 0 ? ping : pong);
        const int64_t ldo = (l == 0) ? ldq : d;
        const size_t sm = L.smem ? size_t(L.rbmax | 1) * d * sizeof(T) : 0;
        cudaFuncSetAttribute(k_hh_form_q<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        k_hh_form_q<T><<<L.nb, kThreads, sm, st>>>(qin, ldqin, L.rows, L.nb, d, V + L.v_off, L.ldv,
                                                    beta + L.beta_off, out, ldo, scratch, L.smem ? 1 : 0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        qin = out;
        ldqin = int(ldo);
    }
    return cudaSuccess;
}

// scratch must hold tsqr_scratch_elems(p) + 2 * max_{l>=1} rows_l * d elements.
template cudaError_t tsqr_factor<double>(const TsqrPlan&, const double*, int64_t, double*, double*, double*,
                                         double*, cudaStream_t);
template cudaError_t tsqr_factor<float>(const TsqrPlan&, const float*, int64_t, float*, float*, float*, float*,
                                        cudaStream_t);
template cudaError_t tsqr_form_q<double>(const TsqrPlan&, const double*, double*, double*, double*, double*,
                                         int64_t, cudaStream_t);
template cudaError_t tsqr_form_q<float>(const TsqrPlan&, const float*, float*, float*, float*, float*, int64_t,
                                        cudaStream_t);

}  // namespace coru_gpu
