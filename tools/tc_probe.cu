// tcgen05 / TMA building-block probe (tooling only): checks each piece of gemm_tc32.cu in isolation.
//  1. TMEM st/ld round trip (32x32b.x32) and the lane mapping of warps 4..7
//  2. one tcgen05.mma kind::tf32, A from TMEM (ts), B from smem MN-major SW128 written by threads
//  3. the same with B K-major SW128 (for comparison)
//  4. 3-D TMA of the pre-tiled X layout into smem (SW128) vs the expected swizzled image
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_1810_07323_b200/csrc/gemm_tc32.cu"

using namespace coru_gpu;

namespace probe {

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout) << 61;
    return d;
}

__device__ __forceinline__ void tc_fb() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fa() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// mode 0: TMEM round trip. mode 1: ts MMA, B MN-major SW128. mode 2: ts MMA, B K-major SW128.
// mode 3: ss MMA, A K-major SW128 + B MN-major SW128.
// A (128 x 8 per K step, 32 K) = a[i][k], B (32 K x 32 N) = b[k][n]; out D 128 x 32.
__global__ void k_probe(int mode, const float* a, const float* b, float* out, uint32_t idesc_override) {
    __shared__ __align__(1024) unsigned char sm[2 * 16384];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    tc_fb();
    __syncthreads();
    tc_fa();
    const uint32_t tmem = slot;
    // B into smem (buffer 1) for N = 32 (one MN atom), K = 32 (4 groups of 8)
    unsigned char* sb = sm + 16384;
    float* sbf = reinterpret_cast<float*>(sb);
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int k = e / 32, n = e % 32;
        if (mode == 1 || mode == 3) {
            // MN-major SW128: row k (128 B = 32 n), 16-B chunk (n/4) ^ (k & 7)
            sbf[k * 32 + (((n >> 2) ^ (k & 7)) << 2) + (n & 3)] = b[k * 32 + n];
        } else if (mode == 2) {
            // K-major SW128: row n (128 B = 32 k), chunk (k/4) ^ (n & 7)
            sbf[n * 32 + (((k >> 2) ^ (n & 7)) << 2) + (k & 3)] = b[k * 32 + n];
        }
    }
    // A into smem (buffer 0) K-major SW128 for mode 3: row i (128 B = 32 k)
    float* saf = reinterpret_cast<float*>(sm);
    if (mode == 3)
        for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
            const int i = e / 32, k = e % 32;
            saf[i * 32 + (((k >> 2) ^ (i & 7)) << 2) + (k & 3)] = a[i * 32 + k];
        }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    // A into TMEM columns 384.. (lane i = row i, column k), warps 4..7
    if (warp >= 4) {
        const int t = threadIdx.x - 128;
        uint32_t v[32];
        for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(a[t * 32 + k]);
        const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
        st32(tmem + lb + 384, v);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    tc_fb();
    __syncthreads();
    tc_fa();
    if (mode >= 1 && threadIdx.x == 32) {
        const uint32_t idesc = idesc_override ? idesc_override
                                              : ((1u << 4) | (2u << 7) | (2u << 10) | ((mode == 2 ? 0u : 1u) << 16) |
                                                 (uint32_t(32 >> 3) << 17) | (uint32_t(128 >> 4) << 24));
        for (int ks = 0; ks < 4; ++ks) {
            uint64_t bd;
            if (mode == 1 || mode == 3) bd = sdesc(smem_u32(sb) + 1024 * ks, 4096, 1024, 2);
            else bd = sdesc(smem_u32(sb) + 32 * ks, 16, 1024, 2);
            const uint32_t acc = ks > 0;
            if (mode == 3) {
                const uint64_t ad = sdesc(smem_u32(sm) + 32 * ks, 16, 1024, 2);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            } else {
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                    "r"(tmem + 384 + 8 * ks), "l"(bd), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar)));
    }
    if (mode >= 1) {
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(&bar)));
    }
    tc_fa();
    if (warp >= 4) {
        const int t = threadIdx.x - 128;
        const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
        uint32_t v[32];
        ld32(tmem + lb + (mode == 0 ? 384 : 0), v);
        for (int j = 0; j < 32; ++j) out[t * 32 + j] = __uint_as_float(v[j]);
    }
    tc_fb();
    __syncthreads();
    if (warp == 2) {
        tc_fa();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

__global__ void k_tma_probe(const __grid_constant__ CUtensorMap tm, float* out, int atoms) {
    __shared__ __align__(1024) unsigned char sm[32 * 1024];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int bytes = 32 * 32 * 4 * atoms;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(bytes));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];\n" ::"r"(smem_u32(sm)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(32), "r"(0), "r"(smem_u32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar)));
    const float* f = reinterpret_cast<const float*>(sm);
    for (int e = threadIdx.x; e < bytes / 4; e += blockDim.x) out[e] = f[e];
}

}  // namespace probe

int main() {
    const int M = 128, K = 32, N = 32;
    std::vector<float> a(M * K), b(K * N), ref(M * N, 0.f), out(M * N);
    for (int i = 0; i < M; ++i)
        for (int k = 0; k < K; ++k) a[i * K + k] = float((i * 3 + k * 7) % 13 - 6);
    for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) b[k * N + n] = float((k * 5 + n * 11) % 17 - 8);
    for (int i = 0; i < M; ++i)
        for (int n = 0; n < N; ++n)
            for (int k = 0; k < K; ++k) ref[i * N + n] += a[i * K + k] * b[k * N + n];
    float *da, *db, *dout;
    cudaMalloc(&da, a.size() * 4);
    cudaMalloc(&db, b.size() * 4);
    cudaMalloc(&dout, out.size() * 4 * 8);
    cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    const char* names[] = {"TMEM st/ld round trip", "ts MMA, B MN-major SW128", "ts MMA, B K-major SW128",
                           "ss MMA, A K-major + B MN-major SW128"};
    for (int mode = 0; mode < 4; ++mode) {
        cudaMemset(dout, 0, out.size() * 4);
        probe::k_probe<<<1, 256>>>(mode, da, db, dout, 0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0, nz = 0;
        double maxerr = 0;
        for (int i = 0; i < M; ++i)
            for (int n = 0; n < N; ++n) {
                const float want = mode == 0 ? a[i * K + n] : ref[i * N + n];
                const float got = out[i * N + n];
                if (got != 0.f) ++nz;
                if (got != want) ++bad;
                maxerr = std::max(maxerr, double(std::abs(got - want)));
            }
        printf("mode %d (%s): %s, wrong %d/%d, nonzero %d, maxerr %g\n", mode, names[mode], cudaGetErrorString(e), bad,
               M * N, nz, maxerr);
        if (bad && mode > 0) {
            printf("  row0 got:");
            for (int n = 0; n < 8; ++n) printf(" %g", out[n]);
            printf("\n  row0 want:");
            for (int n = 0; n < 8; ++n) printf(" %g", ref[n]);
            printf("\n  row1 got:");
            for (int n = 0; n < 8; ++n) printf(" %g", out[N + n]);
            printf("\n  row1 want:");
            for (int n = 0; n < 8; ++n) printf(" %g", ref[N + n]);
            printf("\n");
        }
        if (e != cudaSuccess) return 1;
    }
    // TMA probe: pre-tiled X [atom][k][32] with K = 64, atoms = 2; load k rows 32..63 of both atoms
    {
        const int Kx = 64, atoms = 2;
        std::vector<float> x(atoms * Kx * 32);
        for (size_t e = 0; e < x.size(); ++e) x[e] = float(e);
        float *dx, *dt;
        cudaMalloc(&dx, x.size() * 4);
        cudaMalloc(&dt, 32 * 32 * atoms * 4);
        cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
        CUtensorMap tm;
        const cuuint64_t dims[3] = {32, cuuint64_t(Kx), cuuint64_t(atoms)};
        const cuuint64_t str[2] = {128, cuuint64_t(Kx) * 128};
        const cuuint32_t box[3] = {32, 32, cuuint32_t(atoms)};
        const bool ok = make_map(&tm, dx, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
        probe::k_tma_probe<<<1, 128>>>(tm, dt, atoms);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> got(32 * 32 * atoms);
        cudaMemcpy(got.data(), dt, got.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int at = 0; at < atoms; ++at)
            for (int k = 0; k < 32; ++k)
                for (int c = 0; c < 32; ++c) {
                    const float want = x[(size_t(at) * Kx + 32 + k) * 32 + c];
                    const float g = got[(at * 32 + k) * 32 + ((((c >> 2) ^ (k & 7)) << 2) | (c & 3))];
                    if (g != want) ++bad;
                }
        printf("TMA 3-D pre-tiled X (SW128): map %s, %s, wrong %d/%d; first: %g %g %g %g\n", ok ? "ok" : "FAILED",
               cudaGetErrorString(e), bad, 32 * 32 * atoms, got[0], got[1], got[4], got[32]);
    }
    return 0;
}
