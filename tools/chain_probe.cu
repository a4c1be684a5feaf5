// Hand-off latency probe (tooling only): a chain of 16 warps where warp w waits for warp w-1, does a
// warp reduction, and signals warp w+1 — through (a) named barriers (bar.sync/bar.arrive as in the
// blocked TSQR panel chain) or (b) shared-memory flags (st.release / ld.acquire spin).
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double wsum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k_chain(int mode, int iters, long long* out, double* sink) {
    __shared__ double val[32];
    __shared__ int flag[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double acc = lane;
    if (threadIdx.x < 32) flag[threadIdx.x] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        // warp w > 0 waits for w-1
        if (warp > 0) {
            if (mode == 0) {
                asm volatile("bar.sync %0, %1;\n" ::"r"(1 + ((it * nw + warp - 1) % 15)), "r"(64) : "memory");
            } else {
                int f;
                do {
                    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n" : "=r"(f) : "r"(su(&flag[warp - 1])) : "memory");
                } while (f <= it);
            }
            acc += val[warp - 1];
        } else if (it > 0) {
            if (mode == 0) {
                asm volatile("bar.sync %0, %1;\n" ::"r"(1 + ((it * nw - 1) % 15)), "r"(64) : "memory");
            } else {
                int f;
                do {
                    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n" : "=r"(f) : "r"(su(&flag[nw - 1])) : "memory");
                } while (f < it);
            }
            acc += val[nw - 1];
        }
        acc = wsum(acc) * 1e-3;
        if (lane == 0) val[warp] = acc;
        __syncwarp();
        // signal w+1 (the last warp signals warp 0 of the next iteration)
        if (mode == 0) {
            const int id = 1 + ((it * nw + warp) % 15);
            if (!(warp == nw - 1 && it == iters - 1)) asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(64) : "memory");
        } else {
            if (lane == 0) asm volatile("st.release.cta.shared.b32 [%0], %1;\n" ::"r"(su(&flag[warp])), "r"(it + 1) : "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[mode] = (t1 - t0) / (iters * nw);
    sink[threadIdx.x] = acc;
}

int main() {
    long long* o;
    double* s;
    cudaMallocManaged(&o, 64);
    cudaMalloc(&s, 1024 * 8);
    for (int mode = 0; mode < 2; ++mode) {
        k_chain<<<1, 512>>>(mode, 64, o, s);
        cudaDeviceSynchronize();
        k_chain<<<1, 512>>>(mode, 64, o, s);
        cudaError_t e = cudaDeviceSynchronize();
        printf("%s: %lld cycles per hop (hop = wait + smem read + 5-level fp64 shuffle reduce + signal) [%s]\n",
               mode == 0 ? "named barrier" : "smem flag   ", o[mode], cudaGetErrorString(e));
    }
}
