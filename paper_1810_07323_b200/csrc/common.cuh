// Shared device helpers for the CoR-UTV sm_100a kernels.
#pragma once
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>
#include <cuda_runtime.h>

namespace coru_gpu {

constexpr int kWarp = 32;

// Raise a kernel's dynamic shared-memory limit to the device maximum, once per (kernel, device).
// The attribute is process-global: setting it per launch to the launch's own size races between
// host threads (a concurrent smaller setting makes a larger launch fail), and the limit does not
// affect occupancy — the launch's actual size does.
inline void allow_max_smem(const void* kernel) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert({kernel, dev}).second) return;
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess) v -= int(fa.sharedSizeBytes);  // static smem counts too
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
    cudaGetLastError();  // never leave a stale error for the caller's launch check
}
template <typename K>
inline void allow_max_smem(K* kernel) {
    allow_max_smem(reinterpret_cast<const void*>(kernel));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill: copies `src_bytes` (0..BYTES) and zero-fills the rest of BYTES.
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem_dst, const void* gmem_src, int src_bytes) {
    static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
    if constexpr (BYTES == 16) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem_dst)),
                     "l"(gmem_src), "r"(src_bytes));
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(smem_dst)),
                     "l"(gmem_src), "n"(BYTES), "r"(src_bytes));
    }
}
// 16-byte cp.async with an L2 cache policy (createpolicy): stream A with evict_first so the small,
// re-read operand (the sketch X) stays L2-resident.
__device__ __forceinline__ void cp_async16_hint(void* smem_dst, const void* gmem_src, int src_bytes, uint64_t policy) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(src_bytes), "l"(policy));
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// FP64 tensor-core MMA (DMMA): D[16x8] += A[16x8] * B[8x8], fp64 in/out.
// Fragment layout (g = lane>>2, t = lane&3):
//   a0 (g, t)  a1 (g+8, t)  a2 (g, t+4)  a3 (g+8, t+4)
//   b0 (t, g)  b1 (t+4, g)
//   c0 (g, 2t) c1 (g, 2t+1) c2 (g+8, 2t) c3 (g+8, 2t+1)
__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// Short-latency fp64 reciprocal / reciprocal square root for the latency-bound reflector chains:
// the fp64 MUFU seed (MUFU.RCP64H / MUFU.RSQ64H, from the PTX .approx.ftz.f64 forms) refined by
// Newton steps (DFMA). Measured on B200 (tools/lat2_probe.cu): 54 / 63 cycles dependent latency
// against ~200 for the float-seeded form and ~400 for IEEE division / sqrt; rcp within 1 ulp of
// IEEE, rsqrt within 1.4 ulp. Zero, subnormal, huge and non-finite arguments take the IEEE path.
__device__ __forceinline__ bool mufu64_range(double x) {
    const double a = fabs(x);
    return a > 1e-300 && a < 1e300;
}
__device__ __forceinline__ double fast_rcp(double x) {
    if (!mufu64_range(x)) return 1.0 / x;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double fast_rsqrt(double x) {  // x > 0
    if (!mufu64_range(x)) return 1.0 / sqrt(x);
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    // r <- r (3 - x r^2) / 2, twice (quadratic convergence from the MUFU seed)
    const double h = 0.5 * x;
    r = r * fma(-h * r, r, 1.5);
    r = r * fma(-h * r, r, 1.5);
    return r;
}
__device__ __forceinline__ float fast_rcp(float x) { return 1.0f / x; }
__device__ __forceinline__ float fast_rsqrt(float x) { return rsqrtf(x); }

// make_reflector's scalars (qr.hpp:32-45) for sigma != 0, with two short-latency reciprocals in
// place of the serial IEEE sqrt -> divide -> divide chain:
//   t = x0^2 + sigma, mu = t·rsqrt(t);  v0 = x0 - mu (x0 <= 0) or -sigma/(x0 + mu);
//   beta = 2 v0^2/(sigma + v0^2) = -v0/mu (since sigma = mu^2 - x0^2);
//   rv = 1/v0 = 1/(x0 - mu) or -(x0 + mu)/sigma (the reciprocal of sigma overlaps the rsqrt).
// Every quantity is within a few ulp of the reference's formula.
template <typename T>
__device__ __forceinline__ void reflector_scalars(T x0, T sig, T& mu, T& v0, T& beta, T& rv) {
    const T t = x0 * x0 + sig;
    const T rmu = fast_rsqrt(t);
    const T rsig = fast_rcp(sig);
    mu = t * rmu;
    if (x0 <= T(0)) {
        v0 = x0 - mu;
        rv = fast_rcp(v0);
    } else {
        const T xpm = x0 + mu;
        v0 = -sig * fast_rcp(xpm);
        rv = -xpm * rsig;
    }
    beta = -v0 * rmu;
}

// All-reduce of CPW independent values across the warp with fewer shuffles than CPW butterflies:
// the first log2(CPW) levels reduce-scatter (each lane keeps half of the remaining values), the
// rest finish one value per lane, then the CPW totals are broadcast. 8-byte T: CPW=4 costs 10
// shuffles instead of 20. Deterministic; every lane ends with bitwise identical totals.
template <int CPW, typename T>
__device__ __forceinline__ void warp_allreduce_vec(T (&s)[CPW], int lane) {
    static_assert(CPW == 1 || CPW == 2 || CPW == 4 || CPW == 8, "CPW");
    constexpr int L = CPW == 1 ? 0 : (CPW == 2 ? 1 : (CPW == 4 ? 2 : 3));
    T a[CPW];
#pragma unroll
    for (int i = 0; i < CPW; ++i) a[i] = s[i];
#pragma unroll
    for (int lvl = 0; lvl < L; ++lvl) {
        const int o = 16 >> lvl, half = CPW >> (lvl + 1);
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const T keep = upper ? a[half + i] : a[i];
            const T send = upper ? a[i] : a[half + i];
            a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    T c = a[0];
#pragma unroll
    for (int o = 16 >> L; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        int src = 0;
#pragma unroll
        for (int lvl = 0; lvl < L; ++lvl) src |= ((q >> (L - 1 - lvl)) & 1) << (4 - lvl);
        s[q] = __shfl_sync(0xffffffffu, c, src);
    }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace coru_gpu
