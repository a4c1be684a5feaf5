// pinv of the d x d core for DVariant::approx (corutv.hpp:91-92; svd.hpp:31-187), on one B200.
//
// The reference's Jacobi SVD (svd.hpp:31-134) rotates column pairs in cyclic row order
// (0,1),(0,2),...,(1,2),...: d(d-1)/2 strictly sequential rotations per sweep. Here the pairs of a
// sweep are visited in round-robin (tournament) order instead: each of the d-1 steps of a sweep
// is d/2 disjoint pairs, rotated concurrently, one lane group (4-32 lanes) per pair. Every rotation uses the
// reference's formulas (threshold 1e-14·sqrt(sq_j·sq_k), zeta, t, c, s, recomputed squared norms)
// and the same convergence rule (a sweep without a rotation, at most 60 sweeps); the converged
// factorisation equals the cyclic one up to rounding and the signs of singular-vector pairs,
// neither of which reaches pinv = V·Σ⁺·Uᵀ beyond rounding. Sorting (stable, descending),
// the tolerance d·eps·sigma_1 (svd.hpp:184-187) and the assembly order (matmul(vs, uᵀ),
// r increasing) follow the reference.
//
// Working columns live in shared memory when 2·d² doubles fit (d <= 112 on B200), otherwise in
// the context workspace (L2-resident: 2·520²·8 B = 4.3 MB at C5).
#include <algorithm>
#include <cstdlib>
#include <cfloat>

#include <cooperative_groups.h>

#include "common.cuh"
#include "qrcp.cuh"
#include "svd.cuh"

namespace coru_gpu {
namespace {

constexpr int kJacThreadsMax = 1024;
constexpr int kMaxSweeps = 60;  // svd.hpp:35

// Workspace. After the sweeps, column r of the sorted factorisation is stored contiguously:
//   pinv mode: vs[r] = v(:, src)/sigma (kept r only), ut[r] = a(:, src)/sigma = u(:, r)
//   svd mode:  vs[r] = v(:, src), ut[r] = u(:, r) (0 where sigma == 0, completed later), sig[r]
struct PinvWs {
    double *a, *v, *vs, *ut, *rank, *sq, *sig;  // rank[0] = kept rank; sq: squared norms (grid kernel)
    int *rot, *ord;                             // grid kernel: per-sweep "rotated" flags, sort order
    double *yd, *qp, *rp, *qscr;                // preconditioned pinv: Y (fp64), its QRCP Q and R, scratch
    int64_t* perm;
    __host__ __device__ PinvWs(double* ws, int d) {
        const int64_t dd = int64_t(d) * d;
        a = ws;
        v = a + dd;
        vs = v + dd;
        ut = vs + dd;
        rank = ut + dd;
        sq = rank + 8;
        sig = sq + d;
        rot = reinterpret_cast<int*>(sig + d);
        ord = rot + kMaxSweeps;
        yd = reinterpret_cast<double*>(ws + 4 * dd + 8 + 2 * d + (kMaxSweeps + d + 1) / 2 + 8);
        qp = yd + dd;
        rp = qp + dd;
        perm = reinterpret_cast<int64_t*>(rp + dd);
        qscr = reinterpret_cast<double*>(perm + d);
    }
};

size_t jacobi_smem(int d, bool cols_in_smem) {
    size_t b = size_t(d) * sizeof(double) + size_t(d) * sizeof(int);
    b = (b + 15) / 16 * 16;
    if (cols_in_smem) b += 2 * size_t(d) * d * sizeof(double);
    return b;
}

// Sum over the G lanes of a lane group (xor offsets stay inside aligned groups); every lane of
// the group ends with the same bits.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One CTA. A lane group of G lanes rotates one column pair; a warp carries 32/G pairs, so the
// per-pair scalar work (threshold, zeta, t, c, s) is issued once for 32/G pairs.
// E > 0: the columns live in shared memory and each lane keeps its E entries of the four columns
// of its pair (a_j, a_k, v_j, v_k) in registers for the whole rotation (one load round, one store
// round); E = 0: columns in the global workspace (wide cores), streamed per loop.
template <typename T, int G, int E, int MAXT = (E > 0 ? 512 : kJacThreadsMax)>
__global__ void __launch_bounds__(MAXT, 1)
    k_jacobi_svd(const T* __restrict__ Y, int64_t ldy, int d, double* ws, int cols_in_smem, int* converged_out,
                 int svd_mode) {
    constexpr int kPairsPerWarp = kWarp / G;
    const int kJacThreads = blockDim.x, kJacWarps = kJacThreads >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sq = reinterpret_cast<double*>(smem_raw);
    int* ord = reinterpret_cast<int*>(sq + d);
    const size_t head = (size_t(d) * sizeof(double) + size_t(d) * sizeof(int) + 15) / 16 * 16;
    PinvWs w(ws, d);
    double* a = (E > 0 || cols_in_smem) ? reinterpret_cast<double*>(smem_raw + head) : w.a;
    double* v = a + int64_t(d) * d;
    __shared__ int s_rot;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gl = lane % G;                             // lane within the group
    const int slots = kJacWarps * kPairsPerWarp;
    // column-major working copy (svd.hpp:152-154: a_cm[j·n + i] = a(i, j)) and V = I
    for (int e = tid; e < d * d; e += kJacThreads) {
        const int i = e / d, j = e - i * d;
        a[int64_t(j) * d + i] = double(svd_mode >= 2 ? Y[int64_t(j) * ldy + i] : Y[int64_t(i) * ldy + j]);
        v[int64_t(j) * d + i] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int b = warp * kPairsPerWarp; b < d; b += slots) {  // svd.hpp:38-43 (whole warps join the shuffles)
        const int j = b + lane / G;
        double s = 0.0;
        if (j < d) {
            const double* c = a + int64_t(j) * d;
            for (int i = gl; i < d; i += G) s += c[i] * c[i];
        }
        s = group_sum<G>(s);
        if (j < d && gl == 0) sq[j] = s;
    }

    const int np = d + (d & 1);  // an odd d gets a dummy player
    const int npairs = np / 2, mod = np - 1;
    int converged = 0;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int step = 0; step < mod; ++step) {
            // every lane runs the same trip count so the group shuffles stay converged
            for (int p0 = warp * kPairsPerWarp; p0 < npairs; p0 += slots) {
                const int p = p0 + lane / G;
                // round-robin: position 0 fixed, positions 1..np-1 rotate by `step`
                int x = p - 1 + step, y = np - 2 - p + step;
                x = x >= mod ? x - mod : x;
                y = y >= mod ? y - mod : y;
                x = p == 0 ? 0 : x + 1;
                y += 1;
                const int j = min(x, y), k = max(x, y);
                bool act = p < npairs && k < d;
                const double sqj = act ? sq[j] : 0.0, sqk = act ? sq[k] : 0.0;
                act = act && sqj != 0.0 && sqk != 0.0;  // svd.hpp:50
                double* cj = a + int64_t(act ? j : 0) * d;
                double* ck = a + int64_t(act ? k : 0) * d;
                double* vj = v + int64_t(act ? j : 0) * d;
                double* vk = v + int64_t(act ? k : 0) * d;
                double g = 0.0;
                [[maybe_unused]] double xr[E > 0 ? E : 1], yr[E > 0 ? E : 1], pr[E > 0 ? E : 1], qr[E > 0 ? E : 1];
                if constexpr (E > 0) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int i = gl + e * G;
                        const bool in = act && i < d;
                        xr[e] = in ? cj[i] : 0.0;
                        yr[e] = in ? ck[i] : 0.0;
                        pr[e] = in ? vj[i] : 0.0;
                        qr[e] = in ? vk[i] : 0.0;
                    }
#pragma unroll
                    for (int e = 0; e < E; ++e) g += xr[e] * yr[e];
                } else {
                    if (act)
                        for (int i = gl; i < d; i += G) g += cj[i] * ck[i];
                }
                g = group_sum<G>(g);
                // svd.hpp:53-60. Same rotation, evaluated with one chain of short-latency MUFU-seeded
                // reciprocals: with D = sq_k - sq_j, zeta = D/(2g) and
                //   t = sign(zeta)/(|zeta| + sqrt(1 + zeta^2)) = sign(zeta)·2|g|/(|D| + sqrt(D^2 + 4g^2)),
                // the threshold |g| <= 1e-14·sqrt(sq_j·sq_k) compared in squares, and the reference's
                // "zeta not finite -> skip" as |D| > 2|g|·DBL_MAX.
                const double pjk = sqj * sqk;
                const double ag = fabs(g);
                const bool tiny = (pjk > 1e-280 && pjk < 1e280 && ag < 1e140) ? g * g <= 1e-28 * pjk
                                                                              : ag <= 1e-14 * sqrt(pjk);
                const double D = sqk - sqj;
                act = act && !tiny && !(fabs(D) > 2.0 * ag * DBL_MAX);
                double sj = 0.0, sk = 0.0;
                if (act) {
                    const double qq = D * D + 4.0 * g * g;
                    const double r = mufu64_range(qq) ? qq * fast_rsqrt(qq) : sqrt(qq);
                    const double sgn = (D == 0.0 || (D > 0.0) == (g > 0.0)) ? 1.0 : -1.0;
                    const double t = sgn * (2.0 * ag) * fast_rcp(fabs(D) + r);  // r = inf -> t = 0 (ref :58)
                    const double c = fast_rsqrt(1.0 + t * t);
                    const double s = c * t;
                    if constexpr (E > 0) {
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const int i = gl + e * G;
                            const double nx = c * xr[e] - s * yr[e], ny = s * xr[e] + c * yr[e];
                            const double nv = c * pr[e] - s * qr[e], nw = s * pr[e] + c * qr[e];
                            sj += nx * nx;
                            sk += ny * ny;
                            if (i < d) {
                                cj[i] = nx;
                                ck[i] = ny;
                                vj[i] = nv;
                                vk[i] = nw;
                            }
                        }
                    } else {
                        for (int i = gl; i < d; i += G) {
                            const double xv = cj[i], yv = ck[i];
                            const double nx = c * xv - s * yv, ny = s * xv + c * yv;
                            cj[i] = nx;
                            ck[i] = ny;
                            sj += nx * nx;
                            sk += ny * ny;
                        }
                        for (int i = gl; i < d; i += G) {
                            const double xv = vj[i], yv = vk[i];
                            vj[i] = c * xv - s * yv;
                            vk[i] = s * xv + c * yv;
                        }
                    }
                }
                sj = group_sum<G>(sj);
                sk = group_sum<G>(sk);
                if (act && gl == 0) {
                    sq[j] = sj;
                    sq[k] = sk;
                    s_rot = 1;
                }
            }
            __syncthreads();
        }
        const bool done = s_rot == 0;
        __syncthreads();
        if (done) {
            converged = sweep + 1;  // sweeps used, including the final check sweep
            break;
        }
    }

    // stable sort by descending squared norm (svd.hpp:79-82) as ranks
    for (int j = tid; j < d; j += kJacThreads) {
        const double x = sq[j];
        int r = 0;
        for (int i = 0; i < d; ++i) {
            const double y = sq[i];
            r += (y > x) || (y == x && i < j);
        }
        ord[r] = j;
    }
    __syncthreads();
    const double cut = double(d) * DBL_EPSILON * sqrt(sq[ord[0]]);  // tol·sigma_1 (svd.hpp:172-173)
    // vs(:, r) = v(:, src)·(1/sigma) and ut(r, :) = u(:, src)ᵀ = a(:, src)ᵀ/sigma for kept r
    for (int r = warp; r < d; r += kJacWarps) {
        const int src = ord[r];
        const double sigma = sqrt(sq[src]);
        const double* vc = v + int64_t(src) * d;
        const double* ac = a + int64_t(src) * d;
        if (svd_mode == 1) {  // svd.hpp:84-95
            for (int i = lane; i < d; i += kWarp) {
                w.vs[int64_t(r) * d + i] = vc[i];
                w.ut[int64_t(r) * d + i] = sigma > 0.0 ? ac[i] / sigma : 0.0;
            }
            if (lane == 0) w.sig[r] = sigma;
            continue;
        }
        if (svd_mode == 3) {  // preconditioned svd (svd_square_precond): as mode 2, unscaled, with sigma
            for (int i = lane; i < d; i += kWarp) {
                w.vs[int64_t(r) * d + i] = sigma > 0.0 ? ac[i] / sigma : 0.0;
                w.ut[int64_t(r) * d + i] = vc[i];
            }
            if (lane == 0) w.sig[r] = sigma;
            continue;
        }
        const double inv = sigma > cut ? 1.0 / sigma : 0.0;
        if (inv == 0.0) continue;
        if (svd_mode == 2) {  // X = R^T: V_Y column = P·u'(:, r), U_Y column = Q·v'(:, src) (k_precond_fix)
            for (int i = lane; i < d; i += kWarp) {
                w.vs[int64_t(r) * d + i] = ac[i] / sigma * inv;
                w.ut[int64_t(r) * d + i] = vc[i];
            }
            continue;
        }
        for (int i = lane; i < d; i += kWarp) {
            w.vs[int64_t(r) * d + i] = vc[i] * inv;
            w.ut[int64_t(r) * d + i] = ac[i] / sigma;
        }
    }
    if (tid == 0) {
        int rk = 0;
        while (rk < d && sqrt(sq[ord[rk]]) > cut) ++rk;
        w.rank[0] = double(rk);
        if (converged_out) *converged_out = converged;
    }
}

// Wide cores (columns beyond shared memory, d <= 32·kGridE): the same round-robin sweeps spread
// over a cooperative grid, one warp per pair with the pair's four columns in registers (kGridE
// entries per lane), one grid-wide barrier per step. Columns and norms live in the L2-resident
// workspace and are read with ld.global.cg (other SMs wrote them in the previous step).
constexpr int kGridE = 17;
constexpr int kGridWarps = 4;
template <typename T>
__global__ void __launch_bounds__(kGridWarps * 32)
    k_jacobi_grid(const T* __restrict__ Y, int64_t ldy, int d, double* ws, int* converged_out, int svd_mode) {
    namespace cgs = cooperative_groups;
    cgs::grid_group grid = cgs::this_grid();
    PinvWs w(ws, d);
    double* a = w.a;
    double* v = w.v;
    const int lane = threadIdx.x & 31;
    const int gw = int(blockIdx.x) * kGridWarps + int(threadIdx.x >> 5);
    const int nw = int(gridDim.x) * kGridWarps;
    const int64_t gt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nt = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = gt; e < int64_t(d) * d; e += nt) {
        const int i = int(e / d), j = int(e - int64_t(i) * d);
        a[int64_t(j) * d + i] = double(svd_mode >= 2 ? Y[int64_t(j) * ldy + i] : Y[int64_t(i) * ldy + j]);
        v[int64_t(j) * d + i] = (i == j) ? 1.0 : 0.0;
    }
    if (gt < kMaxSweeps) w.rot[gt] = 0;
    grid.sync();
    for (int j = gw; j < d; j += nw) {  // svd.hpp:38-43
        const double* c = a + int64_t(j) * d;
        double sacc = 0.0;
        for (int i = lane; i < d; i += kWarp) {
            const double x = __ldcg(c + i);
            sacc += x * x;
        }
        sacc = warp_sum(sacc);
        if (lane == 0) w.sq[j] = sacc;
    }
    grid.sync();
    const int np = d + (d & 1), npairs = np / 2, mod = np - 1;
    int converged = 0;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        for (int step = 0; step < mod; ++step) {
            for (int p = gw; p < npairs; p += nw) {
                int x = p - 1 + step, y = np - 2 - p + step;
                x = x >= mod ? x - mod : x;
                y = y >= mod ? y - mod : y;
                x = p == 0 ? 0 : x + 1;
                y += 1;
                const int j = min(x, y), k = max(x, y);
                if (k >= d) continue;
                const double sqj = __ldcg(w.sq + j), sqk = __ldcg(w.sq + k);
                if (sqj == 0.0 || sqk == 0.0) continue;  // svd.hpp:50
                double* cj = a + int64_t(j) * d;
                double* ck = a + int64_t(k) * d;
                double* vj = v + int64_t(j) * d;
                double* vk = v + int64_t(k) * d;
                double xr[kGridE], yr[kGridE], pr[kGridE], qr[kGridE];
                double g = 0.0;
#pragma unroll
                for (int e = 0; e < kGridE; ++e) {
                    const int i = lane + e * kWarp;
                    const bool in = i < d;
                    xr[e] = in ? __ldcg(cj + i) : 0.0;
                    yr[e] = in ? __ldcg(ck + i) : 0.0;
                    pr[e] = in ? __ldcg(vj + i) : 0.0;
                    qr[e] = in ? __ldcg(vk + i) : 0.0;
                }
#pragma unroll
                for (int e = 0; e < kGridE; ++e) g += xr[e] * yr[e];
                g = warp_sum(g);
                const double pjk = sqj * sqk;
                const double ag = fabs(g);
                const bool tiny = (pjk > 1e-280 && pjk < 1e280 && ag < 1e140) ? g * g <= 1e-28 * pjk
                                                                              : ag <= 1e-14 * sqrt(pjk);
                const double D = sqk - sqj;
                if (tiny || fabs(D) > 2.0 * ag * DBL_MAX) continue;  // svd.hpp:53-56
                const double qq = D * D + 4.0 * g * g;
                const double r = mufu64_range(qq) ? qq * fast_rsqrt(qq) : sqrt(qq);
                const double sgn = (D == 0.0 || (D > 0.0) == (g > 0.0)) ? 1.0 : -1.0;
                const double t = sgn * (2.0 * ag) * fast_rcp(fabs(D) + r);
                const double c = fast_rsqrt(1.0 + t * t);
                const double s = c * t;
                double sj = 0.0, sk = 0.0;
#pragma unroll
                for (int e = 0; e < kGridE; ++e) {
                    const int i = lane + e * kWarp;
                    const double nx = c * xr[e] - s * yr[e], ny = s * xr[e] + c * yr[e];
                    const double nv = c * pr[e] - s * qr[e], nq = s * pr[e] + c * qr[e];
                    sj += nx * nx;
                    sk += ny * ny;
                    if (i < d) {
                        __stcg(cj + i, nx);
                        __stcg(ck + i, ny);
                        __stcg(vj + i, nv);
                        __stcg(vk + i, nq);
                    }
                }
                double r2[2] = {sj, sk};
                warp_allreduce_vec<2>(r2, lane);
                if (lane == 0) {
                    __stcg(w.sq + j, r2[0]);
                    __stcg(w.sq + k, r2[1]);
                    __stcg(w.rot + sweep, 1);
                }
            }
            grid.sync();
        }
        if (__ldcg(w.rot + sweep) == 0) {  // read by every thread after the sweep's last barrier
            converged = sweep + 1;
            break;
        }
    }
    // stable descending order (svd.hpp:79-82), then the scaled factors for the assembly
    for (int64_t j = gt; j < d; j += nt) {
        const double x = __ldcg(w.sq + j);
        int rnk = 0;
        for (int i = 0; i < d; ++i) {
            const double y = __ldcg(w.sq + i);
            rnk += (y > x) || (y == x && i < j);
        }
        w.ord[rnk] = int(j);
    }
    grid.sync();
    const double cut = double(d) * DBL_EPSILON * sqrt(__ldcg(w.sq + __ldcg(w.ord)));
    for (int r = gw; r < d; r += nw) {
        const int src = __ldcg(w.ord + r);
        const double sigma = sqrt(__ldcg(w.sq + src));
        const double* vc = v + int64_t(src) * d;
        const double* ac = a + int64_t(src) * d;
        if (svd_mode == 1) {  // svd.hpp:84-95
            for (int i = lane; i < d; i += kWarp) {
                w.vs[int64_t(r) * d + i] = __ldcg(vc + i);
                w.ut[int64_t(r) * d + i] = sigma > 0.0 ? __ldcg(ac + i) / sigma : 0.0;
            }
            if (lane == 0) w.sig[r] = sigma;
            continue;
        }
        if (svd_mode == 3) {
            for (int i = lane; i < d; i += kWarp) {
                w.vs[int64_t(r) * d + i] = sigma > 0.0 ? __ldcg(ac + i) / sigma : 0.0;
                w.ut[int64_t(r) * d + i] = __ldcg(vc + i);
            }
            if (lane == 0) w.sig[r] = sigma;
            continue;
        }
        const double inv = sigma > cut ? 1.0 / sigma : 0.0;
        if (inv == 0.0) continue;
        if (svd_mode == 2) {
            for (int i = lane; i < d; i += kWarp) {
                w.vs[int64_t(r) * d + i] = __ldcg(ac + i) / sigma * inv;
                w.ut[int64_t(r) * d + i] = __ldcg(vc + i);
            }
            continue;
        }
        for (int i = lane; i < d; i += kWarp) {
            w.vs[int64_t(r) * d + i] = __ldcg(vc + i) * inv;
            w.ut[int64_t(r) * d + i] = __ldcg(ac + i) / sigma;
        }
    }
    if (gt == 0) {
        int rk = 0;
        while (rk < d && sqrt(__ldcg(w.sq + __ldcg(w.ord + rk))) > cut) ++rk;
        w.rank[0] = double(rk);
        if (converged_out) *converged_out = converged;
    }
}

// P(i, l) = sum_{r < rank} vs(r, i)·ut(r, l), r increasing (matmul(vs, uᵀ), svd.hpp:180).
constexpr int kAsmTile = 32;
template <typename T>
__global__ void __launch_bounds__(256) k_pinv_assemble(const double* ws, int d, T* P, int64_t ldp) {
    PinvWs w(const_cast<double*>(ws), d);
    __shared__ double sv[kAsmTile][kAsmTile + 1];
    __shared__ double su[kAsmTile][kAsmTile + 1];
    const int rank = int(w.rank[0]);
    const int i0 = blockIdx.y * kAsmTile, l0 = blockIdx.x * kAsmTile;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r0 = 0; r0 < rank; r0 += kAsmTile) {
        for (int rr = ty; rr < kAsmTile; rr += 8) {
            const int r = r0 + rr;
            const bool ok = r < rank;
            sv[rr][tx] = (ok && i0 + tx < d) ? w.vs[int64_t(r) * d + i0 + tx] : 0.0;
            su[rr][tx] = (ok && l0 + tx < d) ? w.ut[int64_t(r) * d + l0 + tx] : 0.0;
        }
        __syncthreads();
        const int rn = min(kAsmTile, rank - r0);
        for (int rr = 0; rr < rn; ++rr) {
            const double u = su[rr][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += sv[rr][ty + 8 * q] * u;
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, l = l0 + tx;
        if (i < d && l < d) P[int64_t(i) * ldp + l] = T(acc[q]);
    }
}


// svd mode, after the sweeps: complete the u columns of zero singular values from the canonical
// basis (svd.hpp:98-121: for each candidate e_i two Gram-Schmidt passes against the earlier
// columns, the largest residual wins, the first on ties), then write U, sigma, V row-major.
template <typename T>
__global__ void __launch_bounds__(1024) k_svd_finalize(double* ws, int d, T* U, int64_t ldu, T* sigma, T* V,
                                                       int64_t ldv) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* cand = reinterpret_cast<double*>(smem_raw);  // [32 warps][d]
    __shared__ double s_res[32];
    __shared__ int s_e[32];
    PinvWs w(ws, d);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* cw = cand + int64_t(warp) * d;
    for (int j = 0; j < d; ++j) {
        if (w.sig[j] > 0.0) continue;  // uniform
        double best = -1.0;
        int be = d;
        for (int e = warp; e < d; e += nw) {
            for (int i = lane; i < d; i += kWarp) cw[i] = (i == e) ? 1.0 : 0.0;
            __syncwarp();
            for (int pass = 0; pass < 2; ++pass)
                for (int c = 0; c < j; ++c) {
                    const double* uc = w.ut + int64_t(c) * d;
                    double dot = 0.0;
                    for (int i = lane; i < d; i += kWarp) dot += cw[i] * uc[i];
                    dot = warp_sum(dot);
                    for (int i = lane; i < d; i += kWarp) cw[i] -= dot * uc[i];
                    __syncwarp();
                }
            double res = 0.0;
            for (int i = lane; i < d; i += kWarp) res += cw[i] * cw[i];
            res = warp_sum(res);
            if (res > best) { best = res; be = e; }  // e increasing: strict > keeps the first
        }
        if (lane == 0) { s_res[warp] = best; s_e[warp] = be; }
        __syncthreads();
        if (warp == 0) {
            double b = lane < nw ? s_res[lane] : -2.0;
            int e = lane < nw ? s_e[lane] : d;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, b, o);
                const int oe = __shfl_xor_sync(0xffffffffu, e, o);
                if (ob > b || (ob == b && oe < e)) { b = ob; e = oe; }
            }
            if (lane == 0) { s_res[0] = b; s_e[0] = e; }
        }
        __syncthreads();
        const int e = s_e[0];
        const double res = s_res[0];
        if (warp == 0) {  // recompute the winner (same arithmetic) straight into u_j
            double* uj = w.ut + int64_t(j) * d;
            for (int i = lane; i < d; i += kWarp) uj[i] = (i == e) ? 1.0 : 0.0;
            __syncwarp();
            for (int pass = 0; pass < 2; ++pass)
                for (int c = 0; c < j; ++c) {
                    const double* uc = w.ut + int64_t(c) * d;
                    double dot = 0.0;
                    for (int i = lane; i < d; i += kWarp) dot += uj[i] * uc[i];
                    dot = warp_sum(dot);
                    for (int i = lane; i < d; i += kWarp) uj[i] -= dot * uc[i];
                    __syncwarp();
                }
            const double nrm = sqrt(res);
            for (int i = lane; i < d; i += kWarp) uj[i] /= nrm;
        }
        __syncthreads();
    }
    for (int64_t e = threadIdx.x; e < int64_t(d) * d; e += blockDim.x) {
        const int i = int(e / d), r = int(e - int64_t(i) * d);
        U[int64_t(i) * ldu + r] = T(w.ut[int64_t(r) * d + i]);
        V[int64_t(i) * ldv + r] = T(w.vs[int64_t(r) * d + i]);
    }
    for (int r = threadIdx.x; r < d; r += blockDim.x) sigma[r] = T(w.sig[r]);
}

// svd_truncate's core (baselines.hpp:14-20): C(i, l) = sum_{r < k} (u(i, r)·sigma_r)·v(l, r), r increasing.
template <typename T>
__global__ void __launch_bounds__(256) k_svd_core(const double* ws, int d, int k, T* C, int64_t ldc) {
    PinvWs w(const_cast<double*>(ws), d);
    __shared__ double su[kAsmTile][kAsmTile + 1];
    __shared__ double sv[kAsmTile][kAsmTile + 1];
    const int i0 = blockIdx.y * kAsmTile, l0 = blockIdx.x * kAsmTile;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r0 = 0; r0 < k; r0 += kAsmTile) {
        for (int rr = ty; rr < kAsmTile; rr += 8) {
            const int r = r0 + rr;
            const bool ok = r < k;
            su[rr][tx] = (ok && i0 + tx < d) ? w.ut[int64_t(r) * d + i0 + tx] * w.sig[r] : 0.0;
            sv[rr][tx] = (ok && l0 + tx < d) ? w.vs[int64_t(r) * d + l0 + tx] : 0.0;
        }
        __syncthreads();
        const int rn = min(kAsmTile, k - r0);
        for (int rr = 0; rr < rn; ++rr) {
            const double vv = sv[rr][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += su[rr][ty + 8 * q] * vv;
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, l = l0 + tx;
        if (i < d && l < d) C[int64_t(i) * ldc + l] = T(acc[q]);
    }
}

// svt's core (rpca.hpp:30-40) on the factors svd_square left in `ws`: R = the leading count of
// sigma_r > delta (the reference's while loop over the non-increasing sigma), then
// C(i, l) = sum_{r < R} (u(i, r)·(sigma_r - delta))·v(l, r), r increasing; R = 0 gives C = 0.
// Block (0, 0) publishes R to *rank_out.
template <typename T>
__global__ void __launch_bounds__(256) k_svt_core(const double* ws, int d, double delta, T* C, int64_t ldc,
                                                  int* rank_out) {
    PinvWs w(const_cast<double*>(ws), d);
    __shared__ double su[kAsmTile][kAsmTile + 1];
    __shared__ double sv[kAsmTile][kAsmTile + 1];
    __shared__ int s_k;
    if (threadIdx.x == 0) {
        int r = 0;
        while (r < d && w.sig[r] > delta) ++r;
        s_k = r;
        if (blockIdx.x == 0 && blockIdx.y == 0 && rank_out) *rank_out = r;
    }
    __syncthreads();
    const int k = s_k;
    const int i0 = blockIdx.y * kAsmTile, l0 = blockIdx.x * kAsmTile;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r0 = 0; r0 < k; r0 += kAsmTile) {
        for (int rr = ty; rr < kAsmTile; rr += 8) {
            const int r = r0 + rr;
            const bool ok = r < k;
            su[rr][tx] = (ok && i0 + tx < d) ? __dmul_rn(w.ut[int64_t(r) * d + i0 + tx], __dsub_rn(w.sig[r], delta)) : 0.0;
            sv[rr][tx] = (ok && l0 + tx < d) ? w.vs[int64_t(r) * d + l0 + tx] : 0.0;
        }
        __syncthreads();
        const int rn = min(kAsmTile, k - r0);
        for (int rr = 0; rr < rn; ++rr) {
            const double vv = sv[rr][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += su[rr][ty + 8 * q] * vv;
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, l = l0 + tx;
        if (i < d && l < d) C[int64_t(i) * ldc + l] = T(acc[q]);
    }
}

// Preconditioned pinv: Y·P = Q·R (QRCP) and the Jacobi SVD of X = R^T = U' Σ V'^T give
// Y = (Q V') Σ (P U')^T, so for every kept r: V_Y(:, r)/σ = P·u'(:, r)/σ (a row permutation) and
// U_Y(:, r) = Q·v'(:, r). One CTA per r.
__global__ void __launch_bounds__(256) k_precond_fix(double* ws, int d) {
    PinvWs w(ws, d);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* x = reinterpret_cast<double*>(smem_raw);
    double* y = x + d;
    const int r = blockIdx.x;
    if (r >= int(w.rank[0])) return;
    double* vr = w.vs + int64_t(r) * d;
    double* ur = w.ut + int64_t(r) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        x[i] = vr[i];
        y[i] = ur[i];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) vr[w.perm[j]] = x[j];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int l = warp; l < d; l += nw) {  // (Q v')(l) = sum_k Q(l, k) v'(k)
        double s = 0.0;
        for (int k = lane; k < d; k += kWarp) s += w.qp[int64_t(l) * d + k] * y[k];
        s = warp_sum(s);
        if (lane == 0) ur[l] = s;
    }
}

template <typename T>
__global__ void k_widen_square(const T* __restrict__ Y, int64_t ldy, int d, double* __restrict__ out) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(d) * d; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / d), j = int(e - int64_t(i) * d);
        out[e] = double(Y[int64_t(i) * ldy + j]);
    }
}
}  // namespace

int64_t pinv_ws_doubles(int d) {
    return 4 * int64_t(d) * d + 8 + 2 * int64_t(d) + (kMaxSweeps + d + 1) / 2 + 8 + 3 * int64_t(d) * d + d +
           qrcp_scratch_elems(d) + 8;
}

template <typename T>
cudaError_t jacobi_run(const T* Y, int64_t ldy, int d, double* ws, int* converged, int max_smem, int svd_mode,
                       cudaStream_t st) {
    const bool in_smem = jacobi_smem(d, true) <= size_t(max_smem);
    static const int jac_variant = getenv("CORU_JACOBI_VARIANT") ? atoi(getenv("CORU_JACOBI_VARIANT")) : 1;
    const size_t smem = jacobi_smem(d, in_smem);
    // G lanes per column pair, at most 8 column entries per lane (register path when the columns
    // fit shared memory); enough warps for the d/2 pairs of a round-robin step
    const int pairs = (d + 1) / 2;
    const int cols = in_smem ? 1 : 0;
    auto launch = [&](auto kern, int G, int max_warps) {
        const int ppw = kWarp / G;
        const int warps = std::min(max_warps, std::max(1, (pairs + ppw - 1) / ppw));
        allow_max_smem(kern);
        kern<<<1, warps * kWarp, smem, st>>>(Y, ldy, d, ws, cols, converged, svd_mode);
    };
    if (in_smem && d <= 32) launch(k_jacobi_svd<T, 4, 8>, 4, 16);
    else if (in_smem && d <= 64) launch(k_jacobi_svd<T, 8, 8>, 8, 16);
    // 64 < d <= 128: 16 lanes per pair fit 32 pairs in 512 threads, so d > 64 takes two rounds per
    // round-robin step; 20 warps (d <= 80, default) run a step in one (d = 80: -6 %); 8 lanes x 16
    // entries (variant 2) is slower (longer per-lane chains).
    else if (in_smem && d <= 80 && jac_variant == 1) launch(k_jacobi_svd<T, 16, 8, 640>, 16, 20);
    else if (in_smem && d <= 128 && jac_variant == 2) launch(k_jacobi_svd<T, 8, 16, 512>, 8, 16);
    else if (in_smem && d <= 128) launch(k_jacobi_svd<T, 16, 8>, 16, 16);
    else if (d <= kWarp * kGridE) {
        // cooperative grid: one warp per pair of a step, every CTA co-resident
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi_grid<T>, kGridWarps * kWarp, 0);
        const int want = (pairs + kGridWarps - 1) / kGridWarps;
        const int blocks = std::max(1, std::min(want, std::max(1, per_sm) * sms));
        int dd = d;
        void* args[] = {(void*)&Y, (void*)&ldy, (void*)&dd, (void*)&ws, (void*)&converged, (void*)&svd_mode};
        cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_jacobi_grid<T>), dim3(blocks),
                                                    dim3(kGridWarps * kWarp), args, 0, st);
        if (e != cudaSuccess) return e;
    } else launch(k_jacobi_svd<T, 32, 0>, 32, 32);
    return cudaGetLastError();
}

template <typename T>
cudaError_t pinv_square(const T* Y, int64_t ldy, int d, T* P, int64_t ldp, double* ws, int* converged, int max_smem,
                        cudaStream_t st) {
    // Preconditioning (default; CORU_PINV_PRECOND=0 turns it off): the one-sided Jacobi of R^T from a
    // column-pivoted QR converges in about half the sweeps of the plain square Jacobi on graded
    // cores (C2 q = 1: 17 -> 8 round-robin sweeps); the pseudo-inverse is the same to rounding.
    static const bool precond = getenv("CORU_PINV_PRECOND") == nullptr || atoi(getenv("CORU_PINV_PRECOND")) != 0;
    cudaError_t e;
    if (precond && d >= 8 && d <= 544) {
        PinvWs w(ws, d);
        k_widen_square<T><<<std::max(1, std::min(148 * 4, (d * d + 255) / 256)), 256, 0, st>>>(Y, ldy, d, w.yd);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = qrcp<double>(w.yd, d, d, w.qp, d, w.rp, d, w.perm, w.qscr, max_smem, st)) != cudaSuccess) return e;
        if ((e = jacobi_run<double>(w.rp, d, d, ws, converged, max_smem, 2, st)) != cudaSuccess) return e;
        k_precond_fix<<<d, 256, 2 * size_t(d) * sizeof(double), st>>>(ws, d);
    } else {
        e = jacobi_run<T>(Y, ldy, d, ws, converged, max_smem, 0, st);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const dim3 grid((d + kAsmTile - 1) / kAsmTile, (d + kAsmTile - 1) / kAsmTile);
    k_pinv_assemble<T><<<grid, 256, 0, st>>>(ws, d, P, ldp);
    return cudaGetLastError();
}

template <typename T>
cudaError_t svd_square(const T* Y, int64_t ldy, int d, T* U, int64_t ldu, T* sigma, T* V, int64_t ldv, double* ws,
                       int* converged, int max_smem, cudaStream_t st) {
    cudaError_t e = jacobi_run<T>(Y, ldy, d, ws, converged, max_smem, 1, st);
    if (e != cudaSuccess) return e;
    const size_t sm = size_t(kWarp) * d * sizeof(double);
    allow_max_smem(k_svd_finalize<T>);
    k_svd_finalize<T><<<1, 1024, sm, st>>>(ws, d, U, ldu, sigma, V, ldv);
    return cudaGetLastError();
}

template <typename T>
cudaError_t svd_factors_precond(const T* Y, int64_t ldy, int d, double* ws, int max_smem, cudaStream_t st) {
    cudaError_t e;
    if (d < 8 || d > 544) return jacobi_run<T>(Y, ldy, d, ws, nullptr, max_smem, 1, st);
    PinvWs w(ws, d);
    k_widen_square<T><<<std::max(1, std::min(148 * 4, (d * d + 255) / 256)), 256, 0, st>>>(Y, ldy, d, w.yd);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = qrcp<double>(w.yd, d, d, w.qp, d, w.rp, d, w.perm, w.qscr, max_smem, st)) != cudaSuccess) return e;
    if ((e = jacobi_run<double>(w.rp, d, d, ws, nullptr, max_smem, 3, st)) != cudaSuccess) return e;
    k_precond_fix<<<d, 256, 2 * size_t(d) * sizeof(double), st>>>(ws, d);
    return cudaGetLastError();
}

template <typename T>
cudaError_t svd_truncate_core(const double* ws, int d, int k, T* C, int64_t ldc, cudaStream_t st) {
    const dim3 grid((d + kAsmTile - 1) / kAsmTile, (d + kAsmTile - 1) / kAsmTile);
    k_svd_core<T><<<grid, 256, 0, st>>>(ws, d, k, C, ldc);
    return cudaGetLastError();
}

template <typename T>
cudaError_t svt_core(const double* ws, int d, double delta, T* C, int64_t ldc, int* rank_out, cudaStream_t st) {
    const dim3 grid((d + kAsmTile - 1) / kAsmTile, (d + kAsmTile - 1) / kAsmTile);
    k_svt_core<T><<<grid, 256, 0, st>>>(ws, d, delta, C, ldc, rank_out);
    return cudaGetLastError();
}

template cudaError_t pinv_square<double>(const double*, int64_t, int, double*, int64_t, double*, int*, int,
                                         cudaStream_t);
template cudaError_t pinv_square<float>(const float*, int64_t, int, float*, int64_t, double*, int*, int,
                                        cudaStream_t);
template cudaError_t svd_square<double>(const double*, int64_t, int, double*, int64_t, double*, double*, int64_t,
                                        double*, int*, int, cudaStream_t);
template cudaError_t svd_truncate_core<double>(const double*, int, int, double*, int64_t, cudaStream_t);

template cudaError_t svd_factors_precond<double>(const double*, int64_t, int, double*, int, cudaStream_t);
template cudaError_t svt_core<double>(const double*, int, double, double*, int64_t, int*, cudaStream_t);

}  // namespace coru_gpu
