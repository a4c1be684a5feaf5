// fp32 A-pass on the 5th-generation tensor cores: tcgen05.mma kind::tf32, 3xTF32 split, TMA-fed.
//
// Replaces, for the fp32 configuration (BASELINE config 5), the three A-passes of corutv —
// matmul(a, c2) (corutv.hpp:55), matmul(at, c1) (corutv.hpp:57, A^T never formed) and the A·Q2 half
// of the projection (corutv.hpp:90) — with the same contract as gemm_f32 (C = op(A)·X, fp32 in/out).
//
// Precision. TF32 keeps 10 mantissa bits; a single TF32 pass would drift ~1e-3 from an fp32 run,
// far outside the fp32 tolerance (SURVEY.md §7 hard part 6). Each operand is split as
// v = hi + lo with hi = rna_tf32(v) (exactly representable) and lo = v - hi (exact in fp32), and
// the tile accumulates lo_A·hi_X + hi_A·lo_X + hi_A·hi_X in the fp32 TMEM accumulator — the
// classic 3xTF32 scheme, whose per-product error is ~2^-21 relative (the dropped lo·lo term and
// the TF32 truncation of the lo parts), i.e. fp32-level.
//
// Data flow per CTA (one 128-row output tile x one N-chunk of nc <= 384 columns; 1 CTA / SM):
//   warp 0      TMA producer: A tile (fp32, raw) + X^hi / X^lo chunk tiles -> smem stage s
//   warps 4..7  converters: row t of the A tile (smem) -> hi/lo -> TMEM columns of stage s
//               (tcgen05.st 32x32b: thread t owns TMEM lane t = output row t); later the epilogue
//   warp 1      MMA issuer (one thread): per K=8 step, 3 (or 6 when nc > 256) tcgen05.mma with
//               A from TMEM ("ts" form) and X from smem (K-major SW128 descriptor); tcgen05.commit
//               frees the stage (smem + TMEM slot) and finally signals the accumulator.
//   warp 2      TMEM allocator (512 columns: accumulator [0, nc), A slots at 384 + 64 s).
// X^hi / X^lo are produced once per pass by k_split_xt, transposed (K-major: row n of the chunk
// holds X(:, n) contiguously; tools/tc_probe.cu showed the MN-major tf32 B operand with the plain
// 128-byte swizzle is not what the tensor core reads, while K-major SW128 is exact). A is read
// exactly once per N-chunk and no A^T is formed: op T loads row-major A tiles as [k][128] and the
// converter reads them down columns.
//
// Deterministic: fixed MMA order; split-K partials reduced in a fixed order (no atomics).
#include <algorithm>
#include <cstring>
#include <mutex>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

constexpr int kTcThreads = 256;
constexpr int kBM = 128;         // output rows per CTA (UMMA M)
constexpr int kBK = 32;          // K per stage (one 128-byte swizzle row of fp32)
constexpr int kAccCols = 384;    // TMEM columns reserved for the accumulator
constexpr int kMaxStages = 2;    // TMEM A slots: 384 + 64 * 2 = 512
constexpr int kATileBytes = kBM * kBK * 4;  // 16 KB
constexpr int kMaxChainKTiles = 128;        // longest fp32 accumulation chain in TMEM: 4096 k, then a flush

// ---- PTX wrappers -------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a pipeline bug traps (launch error) after ~4 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity))
        if (clock64() - t0 > 8000000000LL) __trap();
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), Blackwell version bit 46.
// K-major operand: SBO = byte stride between 8-row groups (1024 for dense 128-byte rows), LBO
// unused by the swizzled K-major form.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

#define CORU_R32(a) a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10], a[11], a[12], a[13], a[14], \
                    a[15], a[16], a[17], a[18], a[19], a[20], a[21], a[22], a[23], a[24], a[25], a[26], a[27],     \
                    a[28], a[29], a[30], a[31]
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}

struct TcArgs {
    int64_t Mo, K;
    int N;        // true columns of C
    int nc;       // columns per N-chunk (multiple of 16, <= kAccCols)
    int n1;       // first MMA's N (<= 256); the second covers nc - n1
    int xboxes;   // TMA boxes per X tile (box rows = nc / xboxes <= 256)
    int nch;      // N-chunks
    int mtiles;
    int stages;
    int kt_per_split;
    float* C;
    int64_t ldc;
    int64_t split_stride;  // > 0: write split partials to C + split * split_stride with ld = N
    int flush_tiles;       // 1: shared memory holds the flush warps' transpose tiles (after the barriers)
};
constexpr int kFlushTileLd = 9;                             // floats per row of a 32 x 8 transpose tile
constexpr int kFlushTileBytes = 4 * 32 * kFlushTileLd * 4;  // four flush warps

template <bool TRANS>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_apass_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
                   const __grid_constant__ CUtensorMap tmXl, const TcArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // 1024-byte alignment for the SW128 atoms
    // 1024-byte alignment for the swizzle atoms, by offsetting the shared pointer itself (an
    // integer round trip would lose the address space and turn every smem access generic)
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int xbytes = p.nc * kBK * 4;                      // one X operand tile per stage
    const int stage_bytes = kATileBytes + 2 * xbytes;       // multiple of 1024
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + p.stages * stage_bytes);
    uint64_t* full = bars;                   // [stages] TMA landed
    uint64_t* conv = bars + kMaxStages;      // [stages] A hi/lo in TMEM
    uint64_t* empty = bars + 2 * kMaxStages; // [stages] MMAs of the stage done (smem + TMEM slot free)
    uint64_t* accf = bars + 3 * kMaxStages;  // accumulator chunk complete
    uint64_t* acce = accf + 1;               // accumulator chunk read back (4 flush warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStages + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int bid = blockIdx.x;
    const int chunk = bid % p.nch;
    bid /= p.nch;
    const int mt = bid % p.mtiles;
    const int split = bid / p.mtiles;
    const int64_t m0 = int64_t(mt) * kBM;
    const int64_t ktiles = (p.K + kBK - 1) / kBK;
    const int64_t kt0 = int64_t(split) * p.kt_per_split;
    const int nk = int((ktiles < kt0 + p.kt_per_split ? ktiles : kt0 + p.kt_per_split) - kt0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 4);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        mbar_init(acce, 4);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmXh)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmXl)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer (whole warp waits, lane 0 issues: the warp stays converged) =====
        for (int i = 0; i < nk; ++i) {
            const int s = i % p.stages;
            if (i >= p.stages) mbar_wait(&empty[s], ((i / p.stages) - 1) & 1);
            if (lane == 0) {
                unsigned char* st = sm + s * stage_bytes;
                mbar_expect_tx(&full[s], uint32_t(stage_bytes));
                const int k0 = int((kt0 + i) * kBK);
                if constexpr (!TRANS)
                    tma_load_2d(st, &tmA, k0, int(m0), &full[s]);
                else
                    tma_load_2d(st, &tmA, int(m0), k0, &full[s]);
                const int br = p.nc / p.xboxes;
                for (int b = 0; b < p.xboxes; ++b) {
                    tma_load_2d(st + kATileBytes + b * br * 128, &tmXh, k0, chunk * p.nc + b * br, &full[s]);
                    tma_load_2d(st + kATileBytes + xbytes + b * br * 128, &tmXl, k0, chunk * p.nc + b * br, &full[s]);
                }
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one thread issues for the CTA) =====
        const uint32_t id1 = idesc_tf32(p.n1);
        const int n2 = p.nc - p.n1;
        const uint32_t id2 = idesc_tf32(n2 > 0 ? n2 : 16);
        for (int i = 0; i < nk; ++i) {
            const int s = i % p.stages;
            const uint32_t ph = (i / p.stages) & 1;
            const bool first = (i % kMaxChainKTiles) == 0;
            if (first && i > 0) mbar_wait(acce, ((i / kMaxChainKTiles) - 1) & 1);  // the last chunk has been read back
            mbar_wait(&full[s], ph);
            mbar_wait(&conv[s], ph);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t xh = smem_u32(sm + s * stage_bytes + kATileBytes);
                const uint32_t xl = xh + xbytes;
                const uint32_t aslot = tmem + kAccCols + 64 * s;
#pragma unroll
                for (int ks = 0; ks < kBK / 8; ++ks) {
                    const uint32_t ahi = aslot + 8 * ks, alo = ahi + 32;
                    const uint32_t acc0 = (!first || ks > 0) ? 1u : 0u;
                    // K-major SW128: rows of 128 B (32 k), 8-row groups 1024 B apart, K step = +32 B
                    const uint64_t bh = sdesc_sw128(xh + 32 * ks, 16, 1024);
                    const uint64_t bl = sdesc_sw128(xl + 32 * ks, 16, 1024);
                    mma_tf32_ts(tmem, alo, bh, id1, acc0);
                    mma_tf32_ts(tmem, ahi, bl, id1, 1u);
                    mma_tf32_ts(tmem, ahi, bh, id1, 1u);
                    if (n2 > 0) {
                        const uint32_t off = p.n1 * 128;
                        const uint64_t bh2 = sdesc_sw128(xh + off + 32 * ks, 16, 1024);
                        const uint64_t bl2 = sdesc_sw128(xl + off + 32 * ks, 16, 1024);
                        mma_tf32_ts(tmem + p.n1, alo, bh2, id2, acc0);
                        mma_tf32_ts(tmem + p.n1, ahi, bl2, id2, 1u);
                        mma_tf32_ts(tmem + p.n1, ahi, bh2, id2, 1u);
                    }
                }
                mma_commit(&empty[s]);
                if ((i % kMaxChainKTiles) == kMaxChainKTiles - 1 || i == nk - 1) mma_commit(accf);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== converters (row t of the tile = TMEM lane t), then the epilogue =====
        const int t = threadIdx.x - 128;
        const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
        const int64_t row = m0 + t;
        const int n0 = chunk * p.nc;
        float* cbase = p.split_stride > 0 ? p.C + split * p.split_stride : p.C;
        const int64_t ldo = p.split_stride > 0 ? int64_t(p.N) : p.ldc;
        float* crow = cbase + row * ldo;
        int nflush = 0;
        for (int i = 0; i < nk; ++i) {
            const int s = i % p.stages;
            const uint32_t ph = (i / p.stages) & 1;
            mbar_wait(&full[s], ph);
            const float* at = reinterpret_cast<const float*>(sm + s * stage_bytes);
            float v[kBK];
            if constexpr (!TRANS) {
                // K-major SW128 tile: row t is 128 bytes, 16-byte chunk c stored at c ^ (t & 7)
#pragma unroll
                for (int c = 0; c < kBK / 4; ++c) {
                    const float4 q = *reinterpret_cast<const float4*>(at + t * kBK + ((c ^ (t & 7)) << 2));
                    v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
                }
            } else {
                // MN-major tile [k][128]: column t
#pragma unroll
                for (int k = 0; k < kBK; ++k) v[k] = at[k * kBM + t];
            }
            uint32_t hi[kBK], lo[kBK];
#pragma unroll
            for (int k = 0; k < kBK; ++k) {
                hi[k] = tf32_rna(v[k]);
                lo[k] = __float_as_uint(v[k] - __uint_as_float(hi[k]));
            }
            if (i >= p.stages) mbar_wait(&empty[s], ((i / p.stages) - 1) & 1);
            tc_fence_after();
            const uint32_t aslot = tmem + lane_base + kAccCols + 64 * s;
            tmem_st32(aslot, hi);
            tmem_st32(aslot + 32, lo);
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
            if ((i % kMaxChainKTiles) == kMaxChainKTiles - 1 || i == nk - 1) {
                // ---- flush: the accumulator of the last <= kMaxChainKTiles k-tiles is added to the
                // output in fp32 round-to-nearest (the tensor core truncates when it accumulates, so
                // one long chain would drift toward zero) and the MMAs restart from zero ----
                if (p.flush_tiles) {
                    // A thread holds 32 columns of ITS row: transposed through a 32 x 8 tile so that
                    // each read-modify-write instruction covers 4 rows x 8 columns = four full
                    // 32-byte sectors (row-per-thread stores touch 32 sectors for 128 bytes). The
                    // output values of a 32-column block are fetched one block ahead (the first
                    // before the accumulator is even complete): L2 latency stays off the chain.
                    float* tile = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(tmem_slot) + 64) +
                                  (warp & 3) * 32 * kFlushTileLd;
                    const int rr = lane >> 3, cc = lane & 7;
                    const int64_t grow0 = m0 + (warp & 3) * 32 + rr;
                    float o[4][8], on[4][8];
                    auto fetch = [&](int cb, float (&dst)[4][8]) {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            const int colc = cb + 8 * g + cc;
                            const bool cok = nflush > 0 && colc < p.nc && n0 + colc < p.N;
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                dst[g][q] = (cok && grow0 + 4 * q < p.Mo) ? cbase[(grow0 + 4 * q) * ldo + n0 + colc] : 0.f;
                        }
                    };
                    fetch(0, o);
                    mbar_wait(accf, nflush & 1);
                    tc_fence_after();
                    for (int cb = 0; cb < p.nc; cb += 32) {
                        uint32_t r[32];
                        tmem_ld32(tmem + lane_base + cb, r);
                        if (cb + 32 < p.nc) fetch(cb + 32, on);
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) tile[lane * kFlushTileLd + j] = __uint_as_float(r[8 * g + j]);
                            __syncwarp();
                            const int colc = cb + 8 * g + cc;
                            const bool cok = colc < p.nc && n0 + colc < p.N;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float v = tile[(4 * q + rr) * kFlushTileLd + cc];
                                if (cok && grow0 + 4 * q < p.Mo) cbase[(grow0 + 4 * q) * ldo + n0 + colc] = o[g][q] + v;
                            }
                            __syncwarp();
                        }
#pragma unroll
                        for (int g = 0; g < 4; ++g)
#pragma unroll
                            for (int q = 0; q < 8; ++q) o[g][q] = on[g][q];
                    }
                } else {
                    mbar_wait(accf, nflush & 1);
                    tc_fence_after();
                    for (int cb = 0; cb < p.nc; cb += 32) {
                        uint32_t r[32];
                        tmem_ld32(tmem + lane_base + cb, r);
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                        if (row < p.Mo) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const int col = n0 + cb + j;
                                if (cb + j < p.nc && col < p.N)
                                    crow[col] = nflush == 0 ? __uint_as_float(r[j]) : crow[col] + __uint_as_float(r[j]);
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(acce);
                ++nflush;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
    }
}

// X (K x N, ld ldx) -> hi / lo parts, transposed: XT[h * nc + n][k] = X[k][h * nc + n] (row
// stride ldk), zero for columns >= N. 32 x 32 tiles through shared memory (coalesced both ways).
__global__ void k_split_xt(const float* __restrict__ X, int64_t ldx, int64_t K, int N, int rows_out, int64_t ldk,
                           float* __restrict__ Xh, float* __restrict__ Xl) {
    __shared__ float tile[32][33];
    const int64_t k0 = int64_t(blockIdx.x) * 32;
    const int n0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    for (int r = ty; r < 32; r += 8) {
        const int64_t k = k0 + r;
        const int n = n0 + tx;
        tile[r][tx] = (k < K && n < N) ? X[k * ldx + n] : 0.f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int n = n0 + r;
        const int64_t k = k0 + tx;
        if (n < rows_out && k < K) {
            const float x = tile[tx][r];
            const float hi = __uint_as_float(tf32_rna(x));
            Xh[int64_t(n) * ldk + k] = hi;
            Xl[int64_t(n) * ldk + k] = x - hi;
        }
    }
}

__global__ void k_reduce_splits_tc(const float* __restrict__ P, int64_t split_stride, int splits, float* __restrict__ C,
                                   int64_t ldc, int64_t rows, int N) {
    const int64_t total = rows * N;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        float s = P[e];
        for (int k = 1; k < splits; ++k) s += P[k * split_stride + e];
        C[(e / N) * ldc + e % N] = s;
    }
}

// ---- host side ----------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
              const cuuint32_t* box, CUtensorMapSwizzle sw) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cuuint32_t(rank), const_cast<void*>(base), dims, strides_bytes, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TcShape {
    int nch, nc, n1, xboxes, stages, splits, mtiles, kt_per_split, flush_tiles;
    size_t smem;
};

TcShape tc_shape(int64_t Mo, int64_t K, int N, int num_sms, int max_smem) {
    TcShape s{};
    const int n16 = (N + 15) / 16 * 16;
    s.nch = (n16 + kAccCols - 1) / kAccCols;
    s.nc = ((n16 / 16 + s.nch - 1) / s.nch) * 16;
    s.n1 = std::min(s.nc, 256);
    s.xboxes = (s.nc + 255) / 256;
    const size_t stage = size_t(kATileBytes) + 2 * size_t(s.nc) * kBK * 4;
    s.stages = int(std::min<size_t>(kMaxStages, (size_t(max_smem) - 1024 - 256) / stage));
    s.smem = 1024 + s.stages * stage + 256;
    s.flush_tiles = s.smem + kFlushTileBytes <= size_t(max_smem) ? 1 : 0;  // not with two 112 KB stages (nc = 384)
    if (s.flush_tiles) s.smem += kFlushTileBytes;
    s.mtiles = int((Mo + kBM - 1) / kBM);
    const int64_t ktiles = (K + kBK - 1) / kBK;
    const int64_t base = int64_t(s.mtiles) * s.nch;
    double best = 1e30;
    int best_s = 1;
    const int max_s = int(std::max<int64_t>(1, std::min<int64_t>(ktiles / 16, 16)));
    // Cost in k-tile times: every CTA pays ~6 k-tiles of fill / flush on top of its share of K,
    // and split partials are written and summed at HBM speed (C5: 13 splits of the 6.9-wave grid
    // looked 1 % better by wave count alone and cost 0.3 ms of reduce per pass — and 1.6x on the
    // K = 8192 products of the sketch over Φ row chunks).
    const double reduce_unit = double(Mo) * double(N) * 8.0 / 9.1e6;
    // (Accuracy does not depend on the split count: the kernel restarts its fp32 TMEM accumulator
    // every kMaxChainKTiles k-tiles — the tensor core truncates when it accumulates, and one
    // 65536-long chain was measured to shrink C5's |t_11| by 3.7e-4 against 13 chains of 5041.)
    for (int sp = 1; sp <= max_s; ++sp) {
        const double waves = std::ceil(double(base * sp) / num_sms);
        const double cost = waves * (double(ktiles) / sp + 6.0) + (sp > 1 ? sp * reduce_unit : 0.0);
        if (cost < best - 1e-9) { best = cost; best_s = sp; }
    }
    s.kt_per_split = int((ktiles + best_s - 1) / best_s);
    s.splits = int((ktiles + s.kt_per_split - 1) / s.kt_per_split);
    return s;
}

}  // namespace

bool gemm_tc32_eligible(int64_t Mo, int64_t K, int N) {
    return N >= 16 && N <= 2 * kAccCols && Mo >= kBM && K >= 4 * kBK;
}

bool gemm_tc32_supported(Op op, const float* A, int64_t lda, int64_t Mo, int64_t K, int N) {
    (void)op;
    if (!encode_fn()) return false;
    if (!gemm_tc32_eligible(Mo, K, N)) return false;
    if ((lda * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0) return false;
    return true;
}

int64_t gemm_tc32_ws_elems(int64_t Mo, int64_t K, int N, int num_sms) {
    const TcShape s = tc_shape(Mo, K, N, num_sms, 227 * 1024);
    const int64_t x = int64_t(s.nch) * s.nc * ((K + 3) / 4 * 4);  // one transposed operand
    return 2 * x + (s.splits > 1 ? int64_t(s.splits) * Mo * N : 0) + 64;
}

cudaError_t gemm_tc32(Op op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C, int64_t ldc,
                      int64_t Mo, int64_t K, int N, float* ws, int num_sms, int max_smem, cudaStream_t st) {
    const TcShape s = tc_shape(Mo, K, N, num_sms, max_smem);
    const int64_t ldk = (K + 3) / 4 * 4;  // TMA row stride must be a multiple of 16 bytes
    const int rows_out = s.nch * s.nc;
    const int64_t xe = int64_t(rows_out) * ldk;
    float* xh = ws;
    float* xl = ws + xe;
    float* part = ws + 2 * xe;
    {
        const dim3 grid(unsigned((K + 31) / 32), unsigned((rows_out + 31) / 32));
        k_split_xt<<<grid, 256, 0, st>>>(X, ldx, K, N, rows_out, ldk, xh, xl);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    CUtensorMap ta, txh, txl;
    if (op == Op::N) {
        const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(Mo)};
        const cuuint64_t str[1] = {cuuint64_t(lda) * 4};
        const cuuint32_t box[2] = {kBK, kBM};
        if (!make_map(&ta, A, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    } else {
        const cuuint64_t dims[2] = {cuuint64_t(Mo), cuuint64_t(K)};
        const cuuint64_t str[1] = {cuuint64_t(lda) * 4};
        const cuuint32_t box[2] = {kBM, kBK};
        if (!make_map(&ta, A, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows_out)};
        const cuuint64_t str[1] = {cuuint64_t(ldk) * 4};
        const cuuint32_t box[2] = {kBK, cuuint32_t(s.nc / s.xboxes)};
        if (!make_map(&txh, xh, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
        if (!make_map(&txl, xl, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    }
    TcArgs a{};
    a.Mo = Mo;
    a.K = K;
    a.N = N;
    a.nc = s.nc;
    a.n1 = s.n1;
    a.xboxes = s.xboxes;
    a.nch = s.nch;
    a.mtiles = s.mtiles;
    a.stages = s.stages;
    a.kt_per_split = s.kt_per_split;
    a.C = s.splits > 1 ? part : C;
    a.ldc = ldc;
    a.split_stride = s.splits > 1 ? Mo * N : 0;
    a.flush_tiles = s.flush_tiles;
    const unsigned grid = unsigned(int64_t(s.nch) * s.mtiles * s.splits);
    if (op == Op::N) {
        allow_max_smem(k_apass_tf32x3<false>);
        k_apass_tf32x3<false><<<grid, kTcThreads, s.smem, st>>>(ta, txh, txl, a);
    } else {
        allow_max_smem(k_apass_tf32x3<true>);
        k_apass_tf32x3<true><<<grid, kTcThreads, s.smem, st>>>(ta, txh, txl, a);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || s.splits == 1) return e;
    const int64_t total = Mo * N;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(num_sms) * 8));
    k_reduce_splits_tc<<<blocks, 256, 0, st>>>(part, Mo * N, s.splits, C, ldc, Mo, N);
    return cudaGetLastError();
}

int gemm_tc32_launches(int64_t Mo, int64_t K, int N, int num_sms) {
    return tc_shape(Mo, K, N, num_sms, 227 * 1024).splits > 1 ? 3 : 2;
}

}  // namespace coru_gpu
