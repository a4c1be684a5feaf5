// pinv of the d x d core for DVariant::approx (corutv.hpp:91-92; svd.hpp:31-187), on one B200.
//
// The reference's Jacobi SVD (svd.hpp:31-134) rotates column pairs in cyclic row order
// (0,1),(0,2),...,(1,2),...: d(d-1)/2 strictly sequential rotations per sweep. Here the pairs of a
// sweep are visited in round-robin (tournament) order instead: each of the d-1 steps of a sweep
// is d/2 disjoint pairs, rotated concurrently, one warp per pair. Every rotation uses the
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
#include <cfloat>

#include "common.cuh"
#include "svd.cuh"

namespace coru_gpu {
namespace {

constexpr int kJacThreadsMax = 1024;
constexpr int kMaxSweeps = 60;  // svd.hpp:35

struct PinvWs {
    double *a, *v, *vs, *ut, *rank;
    __host__ __device__ PinvWs(double* ws, int d) {
        const int64_t dd = int64_t(d) * d;
        a = ws;
        v = a + dd;
        vs = v + dd;
        ut = vs + dd;
        rank = ut + dd;
    }
};

size_t jacobi_smem(int d, bool cols_in_smem) {
    size_t b = size_t(d) * sizeof(double) + size_t(d) * sizeof(int);
    b = (b + 15) / 16 * 16;
    if (cols_in_smem) b += 2 * size_t(d) * d * sizeof(double);
    return b;
}

template <typename T>
__global__ void __launch_bounds__(kJacThreadsMax, 1)
    k_jacobi_svd(const T* __restrict__ Y, int64_t ldy, int d, double* ws, int cols_in_smem, int* converged_out) {
    const int kJacThreads = blockDim.x, kJacWarps = kJacThreads >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sq = reinterpret_cast<double*>(smem_raw);
    int* ord = reinterpret_cast<int*>(sq + d);
    const size_t head = (size_t(d) * sizeof(double) + size_t(d) * sizeof(int) + 15) / 16 * 16;
    PinvWs w(ws, d);
    double* a = cols_in_smem ? reinterpret_cast<double*>(smem_raw + head) : w.a;
    double* v = a + int64_t(d) * d;
    __shared__ int s_rot;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // column-major working copy (svd.hpp:152-154: a_cm[j·n + i] = a(i, j)) and V = I
    for (int e = tid; e < d * d; e += kJacThreads) {
        const int i = e / d, j = e - i * d;
        a[int64_t(j) * d + i] = double(Y[int64_t(i) * ldy + j]);
        v[int64_t(j) * d + i] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int j = warp; j < d; j += kJacWarps) {  // svd.hpp:38-43
        const double* c = a + int64_t(j) * d;
        double s = 0.0;
        for (int i = lane; i < d; i += kWarp) s += c[i] * c[i];
        s = warp_sum(s);
        if (lane == 0) sq[j] = s;
    }

    const int np = d + (d & 1);  // an odd d gets a dummy player
    int converged = 0;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int step = 0; step + 1 < np; ++step) {
            for (int p = warp; p < np / 2; p += kJacWarps) {
                // round-robin: position 0 fixed, positions 1..np-1 rotate by `step`
                const int x = p == 0 ? 0 : (p - 1 + step) % (np - 1) + 1;
                const int y = (np - 2 - p + step) % (np - 1) + 1;
                const int j = min(x, y), k = max(x, y);
                if (k >= d) continue;
                const double sqj = sq[j], sqk = sq[k];
                if (sqj == 0.0 || sqk == 0.0) continue;  // svd.hpp:50
                double* cj = a + int64_t(j) * d;
                double* ck = a + int64_t(k) * d;
                double g = 0.0;
                for (int i = lane; i < d; i += kWarp) g += cj[i] * ck[i];
                g = warp_sum(g);  // butterfly: identical on every lane
                // svd.hpp:53-60 with short-latency reciprocals / square roots (Newton-refined
                // MUFU seeds, ~1 ulp) in place of the serial IEEE divide and sqrt chain
                const double pjk = sqj * sqk;
                if (fabs(g) <= (pjk > 0.0 ? 1e-14 * pjk * fast_rsqrt(pjk) : 0.0)) continue;
                const double zeta = (sqk - sqj) * fast_rcp(2.0 * g);
                if (!isfinite(zeta)) continue;
                const double h = 1.0 + zeta * zeta;
                const double t =
                    isinf(h) ? 0.0 : (zeta >= 0.0 ? 1.0 : -1.0) * fast_rcp(fabs(zeta) + h * fast_rsqrt(h));
                const double c = fast_rsqrt(1.0 + t * t);
                const double s = c * t;
                double sj = 0.0, sk = 0.0;
                for (int i = lane; i < d; i += kWarp) {
                    const double xv = cj[i], yv = ck[i];
                    const double nx = c * xv - s * yv, ny = s * xv + c * yv;
                    cj[i] = nx;
                    ck[i] = ny;
                    sj += nx * nx;
                    sk += ny * ny;
                }
                double* vj = v + int64_t(j) * d;
                double* vk = v + int64_t(k) * d;
                for (int i = lane; i < d; i += kWarp) {
                    const double xv = vj[i], yv = vk[i];
                    vj[i] = c * xv - s * yv;
                    vk[i] = s * xv + c * yv;
                }
                double r2[2] = {sj, sk};
                warp_allreduce_vec<2>(r2, lane);
                if (lane == 0) {
                    sq[j] = r2[0];
                    sq[k] = r2[1];
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
        const double inv = sigma > cut ? 1.0 / sigma : 0.0;
        if (inv == 0.0) continue;
        const double* vc = v + int64_t(src) * d;
        const double* ac = a + int64_t(src) * d;
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

}  // namespace

int64_t pinv_ws_doubles(int d) { return 4 * int64_t(d) * d + 8; }

template <typename T>
cudaError_t pinv_square(const T* Y, int64_t ldy, int d, T* P, int64_t ldp, double* ws, int* converged, int max_smem,
                        cudaStream_t st) {
    const bool in_smem = jacobi_smem(d, true) <= size_t(max_smem);
    const size_t smem = jacobi_smem(d, in_smem);
    allow_max_smem(k_jacobi_svd<T>);
    // one warp per concurrent pair of a round-robin step (d/2 pairs), at most 32 warps
    const int warps = std::min(32, std::max(1, (d + 1) / 2));
    k_jacobi_svd<T><<<1, warps * kWarp, smem, st>>>(Y, ldy, d, ws, in_smem ? 1 : 0, converged);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const dim3 grid((d + kAsmTile - 1) / kAsmTile, (d + kAsmTile - 1) / kAsmTile);
    k_pinv_assemble<T><<<grid, 256, 0, st>>>(ws, d, P, ldp);
    return cudaGetLastError();
}

template cudaError_t pinv_square<double>(const double*, int64_t, int, double*, int64_t, double*, int*, int,
                                         cudaStream_t);
template cudaError_t pinv_square<float>(const float*, int64_t, int, float*, int64_t, double*, int*, int,
                                        cudaStream_t);

}  // namespace coru_gpu
