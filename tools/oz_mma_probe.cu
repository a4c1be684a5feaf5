// Tensor-pipe probe for the Ozaki A-pass (tooling): how many clocks the stage's MMA
// sequence takes when nothing else runs — operands already in shared memory, one CTA per SM, one
// thread issuing, a commit per stage with a bounded number of stages in flight.
//   mode 0: the kernel's stage: A slice s (128 x 32 B, SW32) x stacked X slices 0..6-s, N split at 256
//   mode 1: one N = 256 MMA per "stage" (peak int8 rate of a K = 32 instruction)
//   mode 2: the 28 slice products as 28 separate N = nc MMAs (no stacking)
//   mode 3: like mode 0, but every MMA reads the SAME A slice (operand re-read from one 4 KB block)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc_sw32(uint32_t saddr) {
    uint64_t d = uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t(1) << 16;
    d |= uint64_t(256 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(6) << 61;
    return d;
}
__device__ __forceinline__ uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(su32(bar)), "r"(parity)
                     : "memory");
}

constexpr int kInflight = 4;

__global__ void __launch_bounds__(128, 1) k_probe(int mode, int nc, int stages, long long* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar[kInflight];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 43008 * 2 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0)
        for (int i = 0; i < kInflight; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[i])));
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        for (int i = 0; i < stages; ++i) {
            const int b = i % kInflight;
            if (i >= kInflight) wait(&bar[b], ((i / kInflight) - 1) & 1);
            const uint32_t ab = su32(sm + (i & 1) * 43008), xb = ab + 7 * 4096;
            if (mode == 0 || mode == 3) {
                for (int s = 0; s < 7; ++s) {
                    const int ntot = (7 - s) * nc;
                    const uint64_t ad = sdesc_sw32(ab + (mode == 3 ? 0 : s) * 4096);
                    for (int c0 = 0; c0 < ntot; c0 += 256) {
                        const int n = ntot - c0 < 256 ? ntot - c0 : 256;
                        mma_i8(tmem + s * nc + c0, ad, sdesc_sw32(xb + c0 * 32), idesc_i8(n), (i == 0 && s == 0) ? 0u : 1u);
                    }
                }
            } else if (mode == 1) {
                mma_i8(tmem, sdesc_sw32(ab), sdesc_sw32(xb), idesc_i8(256), i == 0 ? 0u : 1u);
            } else {
                for (int s = 0; s < 7; ++s)
                    for (int t = 0; t + s < 7; ++t)
                        mma_i8(tmem + (s + t) * nc, sdesc_sw32(ab + s * 4096), sdesc_sw32(xb + t * nc * 32), idesc_i8(nc),
                               (i == 0 && s == 0) ? 0u : 1u);
            }
            commit(&bar[b]);
        }
        for (int i = stages; i < stages + kInflight; ++i)
            if (i >= kInflight) wait(&bar[i % kInflight], ((i / kInflight) - 1) & 1);
        if (blockIdx.x == 0) out[0] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int stages = 20000;
    for (int ctas : {1, 148}) {
        for (int mode = 0; mode < 4; ++mode) {
            for (int nc : {64, 48}) {
                if (mode == 1 && nc == 48) continue;
                k_probe<<<ctas, 128, 90 * 1024>>>(mode, nc, stages, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long clk = 0;
                cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
                const double cols = mode == 1 ? 256.0 : 28.0 * nc;
                printf("ctas %3d mode %d nc %2d: %8.1f clk/stage  %7.0f MAC/clk/SM  (%s)\n", ctas, mode, nc, double(clk) / stages,
                       cols * 128 * 32 / (double(clk) / stages), cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
