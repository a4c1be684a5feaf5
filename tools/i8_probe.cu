// tcgen05 kind::i8 building-block probe (tooling only; DESIGN.md §4 "Ozaki A-pass"): pins, on the
// B200, the pieces the int8 tensor-core A-pass (gemm_oz.cu) relies on:
//   1. the smem image of a TMA SWIZZLE_32B load of 32-byte rows (the X digit slices);
//   2. which K-major 32-byte-row smem layout + descriptor the UMMA reads (SW32 vs. no-swizzle
//      core matrices, LBO/SBO roles), for M = 128, N = 64 / 48, K = 32;
//   3. the instruction-descriptor signedness fields (u8/s8 per operand) and s32 accumulation.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout) << 61;
    return d;
}
__device__ __forceinline__ int lay_off(int layout_id, int r, int k) {
    switch (layout_id) {
        case 0: return r * 32 + ((((k >> 4) ^ ((r >> 2) & 1))) << 4) + (k & 15);  // SW32 (bit4 ^= bit7)
        case 1: return ((r >> 3) * 2 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15); // core matrices
        case 2: return r * 32 + k;                                                // plain rows
        default: return 0;
    }
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

// One MMA (or two accumulating) D[128 x N] = A[128 x 32] . B[N x 32]^T, int8 operands written by
// threads in layout `lay` (A and B alike) or B loaded by TMA (use_tma), descriptor (layout_type,
// lbo, sbo). a_signed / b_signed pick the idesc types; D read back as int32.
__global__ void k_mma(const int8_t* a, const int8_t* b, int N, int lay, int ltype, int lbo, int sbo, int atype,
                      int btype, int twice, int use_tma, const __grid_constant__ CUtensorMap tmb, int* out) {
    __shared__ __align__(1024) unsigned char sa[128 * 32];
    __shared__ __align__(1024) unsigned char sb[256 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar[2];
    const int warp = threadIdx.x >> 5;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) sa[lay_off(lay, e / 32, e % 32)] = a[e];
    if (!use_tma)
        for (int e = threadIdx.x; e < N * 32; e += blockDim.x) sb[lay_off(lay, e / 32, e % 32)] = b[e];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = slot;
    if (use_tma && threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar[1])), "r"(N * 32));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                su32(sb)),
            "l"(reinterpret_cast<uint64_t>(&tmb)), "r"(0), "r"(0), "r"(su32(&bar[1]))
            : "memory");
    }
    if (use_tma)
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
                su32(&bar[1])));
    __syncthreads();
    if (threadIdx.x == 32) {
        const uint32_t idesc = (2u << 4) | (uint32_t(atype) << 7) | (uint32_t(btype) << 10) |
                               (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        const uint64_t ad = sdesc(su32(sa), lbo, sbo, ltype);
        const uint64_t bd = sdesc(su32(sb), lbo, sbo, ltype);
        for (int it = 0; it <= twice; ++it) {
            const uint32_t acc = it > 0;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            su32(&bar[0])));
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar[0])));
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp >= 4) {
        const int t = threadIdx.x - 128;
        const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
        for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t v[32];
            ld32(tmem + lb + c0, v);
            for (int j = 0; j < 32 && c0 + j < N; ++j) out[t * N + c0 + j] = int(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

__global__ void k_tma_dump(const __grid_constant__ CUtensorMap tm, unsigned char* out, int bytes) {
    __shared__ __align__(1024) unsigned char sm[8192];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(bytes));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                su32(sm)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(su32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar)));
    for (int e = threadIdx.x; e < bytes; e += blockDim.x) out[e] = sm[e];
}


// ts form: A (128 x 32 int8) from TMEM (lane = row, 8 columns of 4 consecutive k, little-endian),
// B (N x 32, N up to 256) from smem SW32; D at TMEM column dcol.
__global__ void k_mma_ts(const int8_t* a, const int8_t* b, int N, int atype, int btype, int dcol, int* out) {
    __shared__ __align__(1024) unsigned char sb[256 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int e = threadIdx.x; e < N * 32; e += blockDim.x) sb[lay_off(0, e / 32, e % 32)] = b[e];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = slot;
    if (warp >= 4) {
        const int t = threadIdx.x - 128;
        uint32_t w[8];
        for (int c = 0; c < 8; ++c) {
            uint32_t x = 0;
            for (int j = 0; j < 4; ++j) x |= uint32_t(uint8_t(a[t * 32 + 4 * c + j])) << (8 * j);
            w[c] = x;
        }
        const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(tmem + lb + 504),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (threadIdx.x == 32) {
        const uint32_t idesc = (2u << 4) | (uint32_t(atype) << 7) | (uint32_t(btype) << 10) |
                               (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        const uint64_t bd = sdesc(su32(sb), 16, 256, 6);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + dcol),
            "r"(tmem + 504), "l"(bd), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            su32(&bar)));
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp >= 4) {
        const int t = threadIdx.x - 128;
        const uint32_t lb = uint32_t((warp & 3) * 32) << 16;
        for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t v[32];
            ld32(tmem + lb + dcol + c0, v);
            for (int j = 0; j < 32 && c0 + j < N; ++j) out[t * N + c0 + j] = int(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static bool map_u8(CUtensorMap* m, const void* base, int rows, int ld, int box_rows, CUtensorMapSwizzle sw) {
    cuuint64_t dims[2] = {32, cuuint64_t(rows)};
    cuuint64_t str[1] = {cuuint64_t(ld)};
    cuuint32_t box[2] = {32, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    return enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, str, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main() {
    // 1. TMA SW32 image
    {
        const int rows = 64;
        std::vector<unsigned char> g(rows * 32);
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < 32; ++k) g[r * 32 + k] = (unsigned char)((r & 7) * 32 + k);  // row mod 8, byte
        unsigned char *dg, *dout;
        cudaMalloc(&dg, g.size());
        cudaMalloc(&dout, g.size());
        cudaMemcpy(dg, g.data(), g.size(), cudaMemcpyHostToDevice);
        CUtensorMap tm;
        bool ok = map_u8(&tm, dg, rows, 32, rows, CU_TENSOR_MAP_SWIZZLE_32B);
        k_tma_dump<<<1, 128>>>(tm, dout, rows * 32);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<unsigned char> o(g.size());
        cudaMemcpy(o.data(), dout, o.size(), cudaMemcpyDeviceToHost);
        printf("TMA SW32 map=%d err=%s\n", ok, cudaGetErrorString(e));
        int match_sw = 1, match_plain = 1;
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < 32; ++k) {
                const int p_sw = r * 32 + ((((k >> 4) ^ ((r >> 2) & 1))) << 4) + (k & 15);
                if (o[p_sw] != g[r * 32 + k]) match_sw = 0;
                if (o[r * 32 + k] != g[r * 32 + k]) match_plain = 0;
            }
        printf("TMA SW32 image: matches (bit4^=bit7) swizzle: %d, plain: %d\n", match_sw, match_plain);
        for (int r = 0; r < 8; ++r) {
            printf("  smem row %d:", r);
            for (int k = 0; k < 32; k += 16) printf(" [%3d..]", o[r * 32 + k]);
            printf("\n");
        }
    }
    // 2/3. MMA layouts and signedness
    const int M = 128;
    int Ns[2] = {64, 48};
    srand(1);
    for (int ni = 0; ni < 2; ++ni) {
        const int N = Ns[ni];
        std::vector<int8_t> a(M * 32), b(N * 32);
        for (auto& x : a) x = int8_t(rand() & 255);
        for (auto& x : b) x = int8_t(rand() & 255);
        int8_t *da, *db;
        int* dout;
        cudaMalloc(&da, a.size());
        cudaMalloc(&db, b.size());
        cudaMalloc(&dout, M * N * 4);
        cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
        CUtensorMap tmb;
        map_u8(&tmb, db, N, 32, N, CU_TENSOR_MAP_SWIZZLE_32B);
        struct Cfg { int lay, ltype, lbo, sbo; const char* name; };
        Cfg cfgs[] = {{0, 6, 16, 256, "SW32 rows, ltype 6, sbo 256"},
                      {0, 6, 256, 256, "SW32 rows, ltype 6, lbo 256 sbo 256"},
                      {1, 0, 128, 256, "core matrices, none, lbo 128 sbo 256"},
                      {1, 0, 256, 128, "core matrices, none, lbo 256 sbo 128"},
                      {2, 6, 16, 256, "plain rows, ltype 6"}};
        for (int ci = 0; ci < 5; ++ci)
            for (int at = 0; at < 2; ++at)
                for (int bt = 0; bt < 2; ++bt)
                    for (int tw = 0; tw < 2; ++tw)
                        for (int tma = 0; tma < 2; ++tma) {
                            if (tma && cfgs[ci].lay != 0) continue;
                            if ((at != bt || tw) && ci != 0 && ci != 2) continue;
                            cudaMemset(dout, 0, M * N * 4);
                            k_mma<<<1, 256>>>(da, db, N, cfgs[ci].lay, cfgs[ci].ltype, cfgs[ci].lbo, cfgs[ci].sbo, at,
                                              bt, tw, tma, tmb, dout);
                            cudaError_t e = cudaDeviceSynchronize();
                            std::vector<int> o(M * N);
                            cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
                            int bad = 0;
                            for (int i = 0; i < M; ++i)
                                for (int n = 0; n < N; ++n) {
                                    long s = 0;
                                    for (int k = 0; k < 32; ++k) {
                                        const int x = at ? int(a[i * 32 + k]) : int(uint8_t(a[i * 32 + k]));
                                        const int y = bt ? int(b[n * 32 + k]) : int(uint8_t(b[n * 32 + k]));
                                        s += long(x) * y;
                                    }
                                    s *= (tw + 1);
                                    if (o[i * N + n] != int(s)) ++bad;
                                }
                            printf("N=%d %-40s a%s b%s twice=%d tma=%d err=%s bad=%d/%d\n", N, cfgs[ci].name,
                                   at ? "s8" : "u8", bt ? "s8" : "u8", tw, tma, cudaGetErrorString(e), bad, M * N);
                            if (e != cudaSuccess) return 1;
                        }
    }
    // 4. ts form (A from TMEM), N up to 256, D column offsets
    {
        const int Nts[3] = {256, 192, 48};
        const int dcols[3] = {0, 64, 96};
        for (int ni = 0; ni < 3; ++ni) {
            const int N = Nts[ni];
            std::vector<int8_t> a(M * 32), b(N * 32);
            for (auto& x : a) x = int8_t(rand() & 255);
            for (auto& x : b) x = int8_t(rand() & 255);
            int8_t *da, *db;
            int* dout;
            cudaMalloc(&da, a.size());
            cudaMalloc(&db, b.size());
            cudaMalloc(&dout, M * N * 4);
            cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
            cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
            for (int at = 0; at < 2; ++at)
                for (int bt = 0; bt < 2; ++bt) {
                    cudaMemset(dout, 0, M * N * 4);
                    k_mma_ts<<<1, 256>>>(da, db, N, at, bt, dcols[ni], dout);
                    cudaError_t e = cudaDeviceSynchronize();
                    std::vector<int> o(M * N);
                    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
                    int bad = 0;
                    for (int i = 0; i < M; ++i)
                        for (int n = 0; n < N; ++n) {
                            long sacc = 0;
                            for (int k = 0; k < 32; ++k) {
                                const int x = at ? int(a[i * 32 + k]) : int(uint8_t(a[i * 32 + k]));
                                const int y = bt ? int(b[n * 32 + k]) : int(uint8_t(b[n * 32 + k]));
                                sacc += long(x) * y;
                            }
                            if (o[i * N + n] != int(sacc)) ++bad;
                        }
                    printf("ts N=%d dcol=%d a%s b%s err=%s bad=%d/%d\n", N, dcols[ni], at ? "s8" : "u8", bt ? "s8" : "u8",
                           cudaGetErrorString(e), bad, M * N);
                    if (e != cudaSuccess) return 1;
                }
        }
    }
    return 0;
}
