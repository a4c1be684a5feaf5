// FP64 A-pass on the 5th-generation INT8 tensor cores: tcgen05.mma kind::i8, Ozaki-scheme
// emulation of the fp64 product, TMA-fed, accumulators in TMEM.
//
// Replaces, for the fp64 configurations, the A-passes of corutv — matmul(a, c2) (corutv.hpp:55),
// matmul(at, c1) (corutv.hpp:57, A^T never formed) and the A·Q2 half of the projection
// (corutv.hpp:90) — with the gemm_f64 contract (C = op(A)·X, fp64 in/out, deterministic).
//
// Why. B200's FP64 path (DMMA) peaks at ~36 TFLOP/s, so a d = 110 A-pass over 3.2 GB (C3) is
// compute-bound at 2.5 ms while its HBM time is 0.5 ms. The INT8 tensor cores run 4.5 POPS.
// Ozaki's scheme splits each fp64 operand into 8-bit digit slices against a per-row (A) and
// per-column (X) power-of-two scale; every slice product is EXACT in the int32 accumulator, and
// the products are recombined in fp64. With S = 7 slices (55-bit significands) and the
// triangular truncation s + t <= 6 (28 slice products) the result carries ~2^-55 relative error
// against row-max x column-max, i.e. fp64-level accuracy (tests/test_gpu_oz.py measures it against
// an extended-precision product next to the DMMA kernel's).
//
// Number format. Row i of op(A) has E_i with max_k |a_ik| < 2^E_i (gemm_oz_exponents, once per
// decomposition: A does not change between passes). V_ik = rint(a_ik · 2^(54 - E_i)) is an
// int64 with |V| < 2^54, written in balanced base 256: V + C with C = 0x0080808080808080 has
// byte 6 = the top digit (signed, |.| <= 64) and bytes 5..0 = the other digits + 128, so
// XOR 0x80 turns them into signed digits in [-128, 127] — V = sum_s d_s · 2^(8(6 - s)) with no
// carry loop; the conversion is one F2I, a 64-bit add and byte permutes. Signed (zero-mean)
// digits keep the dropped low-order part of each product unbiased, so it grows like sqrt(K), not
// K. X is split the same way per column j (F_j) by k_oz_split_x. a·x = V·W·2^(E_i + F_j - 108);
// level L = s + t collects the slice products of weight 2^(8(12 - L)); levels 0..6 are
// accumulated (int32, nc TMEM columns each), the rest (< 2^-52 relative, zero-mean) dropped.
// int32 headroom: a level sums <= 7 products of <= 2^14 per k, so accumulators are flushed to fp64
// every kOzChunkStages x 32 = 16384 k (< 2^31 / (7·2^14)).
//
// MMA shape. All digits are s8, so the slice products of one A slice s against X slices
// 0..6-s are ONE stacked operation: B = the X slices stacked along N (contiguous in shared memory),
// D = TMEM columns [s·nc, 7·nc) = levels s..6 — a level-L block receives slice t = L - s exactly
// where it belongs. 28 products per stage become 9-10 tcgen05.mma of N <= 256 (small-N MMAs are
// issue-bound on the tensor pipe).
//
// Data flow per CTA (one 128-row tile of op(A) x one N-chunk of nc <= 64 columns; 1 CTA / SM;
// the nch CTAs of a row tile are adjacent in the grid so A comes from DRAM once and L2 after):
//   warp 0      TMA producer: fp64 A tile (128 x 32) -> fp64 ring (kOzF stages ahead)
//   warp 3      TMA producer: the 7 X digit slices of the chunk (one 3-D box: 7 x nc x 32 int8,
//               SWIZZLE_32B, slices stacked) -> int8 ring
//   warps 4..19 converters: thread (row r, k-quarter kq) reads 8 fp64 of its row (op N: swizzled
//               K-major tile; op T: a column of the [k][m] tile — A^T is never formed), scales,
//               F2I, permutes bytes into the 7 A slices (K-major SW32 rows of 32 B) of the int8
//               ring (16 warps: four per scheduler hide the conversion latencies better than two,
//               1.70 vs 1.83 ms per C3 pass); at each flush they read the 7 level accumulators
//               back (tcgen05.ld) and add
//               sum_L acc_L 2^(-8L) · 2^(E_i + F_j - 12) into the fp64 output (own rows, fixed
//               order: deterministic)
//   warp 1      MMA issuer: per stage and A slice s one stacked tcgen05.mma (M = 128, K = 32,
//               N = (7 - s)·nc split at 256), s8 x s8, A and B from shared memory descriptors
//   warp 2      TMEM allocator
// Split-K (op T: K = m rows of A) writes per-split fp64 partials summed in a fixed order.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gemm.cuh"

namespace coru_gpu {

namespace {

#ifndef CORU_OZ_KQ
#define CORU_OZ_KQ 4
#endif
constexpr int kOzKQ = CORU_OZ_KQ;      // k-groups per stage row (2 or 4): a converter thread takes 32 / kOzKQ doubles
constexpr int kOzEPT = 32 / kOzKQ;     // elements per converter thread and stage
constexpr int kOzConvWarps = 4 * kOzKQ;  // converter warps: kOzKQ per TMEM lane quadrant
constexpr int kOzThreads = 128 + 32 * kOzConvWarps;
constexpr int kOzBM = 128;
constexpr int kOzBK = 32;              // k per stage = one UMMA K step of int8
constexpr int kOzS = 7;                // digit slices per operand
constexpr int kOzNcMax = 64;           // columns per N-chunk
constexpr int kOzMaxChunks = 4;        // N <= 256
#ifndef CORU_OZ_F
#define CORU_OZ_F 3
#endif
#ifndef CORU_OZ_I
#define CORU_OZ_I 3
#endif
constexpr int kOzF = CORU_OZ_F;        // fp64 ring stages (96 KB of A in flight per SM)
constexpr int kOzI = CORU_OZ_I;        // int8 ring stages (converters + X slices -> MMA)
constexpr int kOzChunkStages = 512;    // flush interval (stages): 16384 k
constexpr int kOzF64Bytes = kOzBM * kOzBK * 8;                  // 32 KB
constexpr int kOzASlice = kOzBM * kOzBK;                        // 4 KB
constexpr int kOzXSlice = kOzNcMax * kOzBK;                     // 2 KB (slots stack at nc rows)
constexpr int kOzIStage = kOzS * (kOzASlice + kOzXSlice);       // 42 KB
constexpr int kOzXOff = kOzS * kOzASlice;                       // X slices after the A slices
constexpr int kOzSmem = 1024 + kOzF * kOzF64Bytes + kOzI * kOzIStage + 256;

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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// Shared -> global tensor store (bulk async group of the issuing thread).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, int c0, int c1, int c2, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* tm) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// K-major SWIZZLE_32B operand: rows of 32 bytes (32 int8 k), 8-row groups 256 B apart; the
// 16-byte half of row r holding k in [16c, 16c + 16) sits at half c ^ ((r >> 2) & 1).
__device__ __forceinline__ uint64_t sdesc_sw32(uint32_t saddr) {
    uint64_t d = uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t(1) << 16;                  // LBO (unused by swizzled K-major)
    d |= uint64_t(256 >> 4) << 32;           // SBO: 8 rows x 32 B
    d |= uint64_t(1) << 46;                  // Blackwell descriptor version
    d |= uint64_t(6) << 61;                  // SWIZZLE_32B
    return d;
}
// Instruction descriptor, kind::i8: D s32, A and B s8, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kOzBM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}

// 2^e as a double for e in [-1022, 1023].
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double(int64_t(e + 1023) << 52); }

// Balanced base-256 digits of the int64 w (|w| < 2^54): bytes of w + C, the low six XOR 0x80.
constexpr unsigned long long kOzBias = 0x0000808080808080ull;

// Tooling alternative (CORU_OZ_MAGIC) to F2I.S64.F64: rint(t) + kOzBias for |t| < 2^54,
// bit-identical to (unsigned long long)__double2ll_rn(t) + kOzBias, on the FP64 pipe only — measured
// SLOWER on B200 than the XU conversion (1.93 vs 1.70 ms per C3 pass), kept for the A/B.
// H = rint(t·2^-28) and L = rint(t - H·2^28) by the add-magic-constant trick
// (1.5·2^52 puts the rounded integer in the low mantissa word; both steps exact, ties keep their
// parity because H·2^28 is even), four FP64-pipe operations and a few integer ones.
// t = x·sc (sc a power of two, so x·sc and x·sc·2^-28 are exact): um = rn(t·2^-28 + M), H = um - M,
// c = M - H·2^28 (exact: a multiple of 2^28 below 2^55), lm = rn(t + c) = rn((t - H·2^28) + M).
__device__ __forceinline__ unsigned long long oz_round_biased(double x, double sc, double sc28) {
    constexpr double M = 6755399441055744.0;  // 1.5 · 2^52
    const double um = __fma_rn(x, sc28, M);
    const double hr = __dadd_rn(um, -M);
    const double c = __fma_rn(hr, -0x1p28, M);
    const double lm = __fma_rn(x, sc, c);
    const long long v = (static_cast<long long>(__double2loint(um)) << 28) + static_cast<long long>(__double2loint(lm));
    return static_cast<unsigned long long>(v) + kOzBias;
}

// Exponent E with max |x| < 2^E from the largest biased exponent field be of a group (0 for an
// all-zero group); clamped so the conversion scale 2^(55 - E) stays finite.
__host__ __device__ __forceinline__ int oz_exp_from_biased(int be) {
    if (be <= 0) return 0;                      // all zero (or denormal): any scale works
    const int e = be - 1022;                    // x = m·2^(be-1023), m in [1,2) -> x < 2^(be-1022)
    return e < -960 ? -960 : (e > 1022 ? 1022 : e);
}

struct OzArgs {
    int64_t Mo, K;
    int N;
    int nch;
    int n0[kOzMaxChunks], nc[kOzMaxChunks];
    int xrows;          // rows per slice in the X slice buffer
    int nc_a;           // chunk width served by tmXa (the others use tmXb)
    int mtiles;
    int kt_per_split;   // stages per split
    double* C;
    int64_t ldc;
    int64_t split_stride;  // > 0: split partials at C + split * split_stride, ld = N
    const int* eA;      // per output row: E_i
    const int* eX;      // per column of X: F_j
};

// STORE (op N only): the chunk-0 CTA of every row tile also writes the A digit slices it has just
// built to the PN digit planes (tmP, the map k_apass_ozp loads them with: the stage image in shared
// memory IS the box), so that the later op-N passes of the decomposition run on k_apass_ozp
// without a conversion pass of their own (capi.cu oz_prepare, "hybrid").
template <bool TRANS, bool STORE>
__global__ void __launch_bounds__(kOzThreads, 1)
    k_apass_oz(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXa,
               const __grid_constant__ CUtensorMap tmXb, const __grid_constant__ CUtensorMap tmP,
               const __grid_constant__ OzArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // 1024-byte alignment for the swizzle atoms, by offsetting the shared pointer itself (an
    // integer round trip would lose the address space and turn every smem access generic)
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* fring = sm;
    unsigned char* iring = sm + kOzF * kOzF64Bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(iring + kOzI * kOzIStage);
    uint64_t* f_full = bars;
    uint64_t* f_empty = bars + kOzF;
    uint64_t* x_full = bars + 2 * kOzF;
    uint64_t* a_full = x_full + kOzI;
    uint64_t* i_empty = a_full + kOzI;
    uint64_t* acc_full = i_empty + kOzI;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int bid = blockIdx.x;
    const int chunk = bid % p.nch;
    bid /= p.nch;
    const int mt = bid % p.mtiles;
    const int split = bid / p.mtiles;
    const int n0 = p.n0[chunk], nc = p.nc[chunk];
    const int64_t m0 = int64_t(mt) * kOzBM;
    const int64_t ktiles = (p.K + kOzBK - 1) / kOzBK;
    const int64_t kt0 = int64_t(split) * p.kt_per_split;
    const int nk = int((ktiles < kt0 + p.kt_per_split ? ktiles : kt0 + p.kt_per_split) - kt0);

    const bool storing = STORE && chunk == 0;  // an int8 slot is then released by the MMAs AND the store
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kOzF; ++s) {
            mbar_init(&f_full[s], 1);
            mbar_init(&f_empty[s], kOzConvWarps);
        }
        for (int s = 0; s < kOzI; ++s) {
            mbar_init(&x_full[s], 1);
            mbar_init(&a_full[s], kOzConvWarps);
            mbar_init(&i_empty[s], storing ? 2 : 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, kOzConvWarps);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(nc == p.nc_a ? &tmXa : &tmXb))
                     : "memory");
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
        // ===== TMA producer: fp64 A tiles, F stages ahead of the converters =====
        for (int i = 0; i < nk; ++i) {
            const int fs = i % kOzF;
            const int k0 = int((kt0 + i) * kOzBK);
            if (i >= kOzF) mbar_wait(&f_empty[fs], ((i / kOzF) - 1) & 1);
            if (lane == 0) {
                unsigned char* dst = fring + fs * kOzF64Bytes;
                mbar_expect_tx(&f_full[fs], uint32_t(kOzF64Bytes));
                if constexpr (!TRANS) {
                    tma_load_2d(dst, &tmA, k0, int(m0), &f_full[fs]);
                    tma_load_2d(dst + kOzF64Bytes / 2, &tmA, k0 + 16, int(m0), &f_full[fs]);
                } else {
                    tma_load_2d(dst, &tmA, int(m0), k0, &f_full[fs]);
                }
            }
            __syncwarp();
        }
    } else if (warp == 3) {
        // ===== TMA producer: X digit slices into the int8 ring (paced by the MMAs) =====
        for (int i = 0; i < nk; ++i) {
            const int is = i % kOzI;
            const int k0 = int((kt0 + i) * kOzBK);
            if (i >= kOzI) mbar_wait(&i_empty[is], ((i / kOzI) - 1) & 1);
            if (lane == 0) {
                // the chunk's 7 slices stacked: slot t at t·nc rows (one 3-D box)
                unsigned char* xs = iring + is * kOzIStage + kOzXOff;
                mbar_expect_tx(&x_full[is], uint32_t(kOzS * nc * kOzBK));
                tma_load_3d(xs, nc == p.nc_a ? &tmXa : &tmXb, k0, n0, 0, &x_full[is]);
            }
            __syncwarp();
        }
    } else if (STORE && warp == 2) {
        // ===== plane store: the A slices of each stage -> PN, one stage behind =====
        if (storing) {
            if (lane == 0) prefetch_tensormap(&tmP);
            for (int i = 0; i < nk; ++i) {
                const int is = i % kOzI;
                mbar_wait(&a_full[is], (i / kOzI) & 1);
                if (lane == 0) {
                    tma_store_3d(&tmP, int((kt0 + i) * kOzBK), int(m0), 0, iring + is * kOzIStage);
                    if (i > 0) {
                        tma_store_wait_read<1>();  // the previous stage's slices have left shared memory
                        mbar_arrive(&i_empty[(i - 1) % kOzI]);
                    }
                }
                __syncwarp();
            }
            if (lane == 0) {
                tma_store_wait_read<0>();
                mbar_arrive(&i_empty[(nk - 1) % kOzI]);
                asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        for (int i = 0; i < nk; ++i) {
            const int is = i % kOzI;
            const uint32_t ph = (i / kOzI) & 1;
            const int ci = i / kOzChunkStages;
            const bool first = (i % kOzChunkStages) == 0;
            if (first && ci > 0) mbar_wait(acc_empty, (ci - 1) & 1);
            mbar_wait(&x_full[is], ph);
            mbar_wait(&a_full[is], ph);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t ab = smem_u32(iring + is * kOzIStage);
                const uint32_t xb = ab + kOzXOff;
#pragma unroll
                for (int s = 0; s < kOzS; ++s) {
                    // A slice s x X slices 0..6-s -> levels s..6 (TMEM columns [s·nc, 7·nc))
                    const int ntot = (kOzS - s) * nc;
                    const uint64_t ad = sdesc_sw32(ab + s * kOzASlice);
                    for (int c0 = 0; c0 < ntot; c0 += 256) {
                        const int n = ntot - c0 < 256 ? ntot - c0 : 256;
                        mma_i8(tmem + uint32_t(s * nc + c0), ad, sdesc_sw32(xb + c0 * kOzBK), idesc_i8(n),
                               (first && s == 0) ? 0u : 1u);
                    }
                }
                mma_commit(&i_empty[is]);
                if ((i % kOzChunkStages) == kOzChunkStages - 1 || i == nk - 1) mma_commit(acc_full);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== converters, then the flushes =====
        // warp cw: TMEM lane quadrant q = cw & 3 (= warp % 4, the lanes tcgen05.ld may touch),
        // k-group kq = cw >> 2: thread (row r, kq) converts the kOzEPT doubles k = kq·EPT .. of its row.
        const int cw = warp - 4, q = cw & 3, kq = cw >> 2;
        const int r = q * 32 + lane;
        const int64_t row = m0 + r;
        const int E = row < p.Mo ? p.eA[row] : 0;
        const double sc = pow2(54 - E), sc28 = pow2(26 - E);
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const int k_first = kq * kOzEPT;        // first k of this thread within the stage
        int nflush = 0;
        for (int i = 0; i < nk; ++i) {
            const int fs = i % kOzF, is = i % kOzI;
            mbar_wait(&f_full[fs], (i / kOzF) & 1);
            double v[kOzEPT];
            const unsigned char* ft = fring + fs * kOzF64Bytes;
            if constexpr (!TRANS) {
                // box k/16: 128 rows x 16 doubles, SW128: 16-byte chunk c of row r at c ^ (r & 7)
                const unsigned char* rowp = ft + (k_first >> 4) * (kOzF64Bytes / 2) + r * 128;
                const int c0 = (k_first & 15) >> 1;
#pragma unroll
                for (int c = 0; c < kOzEPT / 2; ++c) {
                    const double2 d2 = *reinterpret_cast<const double2*>(rowp + (((c0 + c) ^ (r & 7)) << 4));
                    v[2 * c] = d2.x;
                    v[2 * c + 1] = d2.y;
                }
            } else {
                const double* col = reinterpret_cast<const double*>(ft) + k_first * kOzBM + r;
#pragma unroll
                for (int j = 0; j < kOzEPT; ++j) v[j] = col[j * kOzBM];
            }
            uint32_t lo[kOzEPT], hi[kOzEPT];
#pragma unroll
            for (int j = 0; j < kOzEPT; ++j) {
#if defined(CORU_OZ_MAGIC)                     // tooling: FP64-pipe rounding (measured slower than F2I: 1.93 vs 1.70 ms)
                const unsigned long long w = oz_round_biased(v[j], sc, sc28);
#else
                (void)sc28;
                const unsigned long long w = (unsigned long long)__double2ll_rn(v[j] * sc) + kOzBias;
#endif
                lo[j] = uint32_t(w);
                hi[j] = uint32_t(w >> 32);
            }
            // The fp64 slot is released once every lane has consumed its values: an arrive right
            // after the loads were ISSUED let the next TMA fill overwrite the slot under a lane's
            // outstanding load (seen with 16 converter warps: scattered wrong rows, tools/oz_stress.py).
            __syncwarp();
            if (lane == 0) mbar_arrive(&f_empty[fs]);
            if (i >= kOzI) mbar_wait(&i_empty[is], ((i / kOzI) - 1) & 1);
            // row r of a slice: 32 bytes, the 16-byte half holding k in [16c, 16c+16) at c ^ ((r >> 2) & 1)
            unsigned char* as = iring + is * kOzIStage + r * 32 + ((((k_first >> 4) ^ ((r >> 2) & 1)) << 4) | (k_first & 15));
#pragma unroll
            for (int s = 0; s < kOzS; ++s) {
                const int b = 6 - s;  // byte of V holding slice s
                uint32_t w4[kOzEPT / 4];
#pragma unroll
                for (int g = 0; g < kOzEPT / 4; ++g) {
                    const uint32_t* src = b < 4 ? lo : hi;
                    const uint32_t bb = uint32_t(b & 3);
                    const uint32_t t01 = __byte_perm(src[4 * g], src[4 * g + 1], bb | ((bb + 4) << 4));
                    const uint32_t t23 = __byte_perm(src[4 * g + 2], src[4 * g + 3], bb | ((bb + 4) << 4));
                    w4[g] = __byte_perm(t01, t23, 0x5410) ^ (s == 0 ? 0u : 0x80808080u);
                }
                if constexpr (kOzEPT == 16)
                    *reinterpret_cast<uint4*>(as + s * kOzASlice) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                else
                    *reinterpret_cast<uint2*>(as + s * kOzASlice) = make_uint2(w4[0], w4[1]);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_full[is]);
            if ((i % kOzChunkStages) == kOzChunkStages - 1 || i == nk - 1) {
                // ---- flush: fp64 += sum_L acc_L 2^(-8L) · 2^(E + F_j - 12) ----
                mbar_wait(acc_full, nflush & 1);
                tc_fence_after();
                double* out;
                if (p.split_stride > 0)
                    out = p.C + split * p.split_stride + row * p.N;
                else
                    out = p.C + row * p.ldc;
                for (int cb = kq * 8; cb < nc; cb += 8 * kOzKQ) {
                    uint32_t acc[kOzS][8];
#pragma unroll
                    for (int L = 0; L < kOzS; ++L) tmem_ld8(tmem + lane_base + uint32_t(L * nc + cb), acc[L]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int col = n0 + cb + j;
                        double s = double(int(acc[kOzS - 1][j]));
#pragma unroll
                        for (int L = kOzS - 2; L >= 0; --L) s = fma(s, 0.00390625, double(int(acc[L][j])));
                        if (row < p.Mo && col < p.N && cb + j < nc) {
                            const int ex = E + p.eX[col] - 12;
                            // s · 2^ex in two exact steps (ex may leave the normal range of one factor)
                            const double val = (s * pow2(ex >> 1)) * pow2(ex - (ex >> 1));
                            out[col] = nflush == 0 ? val : out[col] + val;
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(acc_empty);
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

// ---- pre-converted digit planes ----------------------------------------------------------------
// A decomposition streams the same A 2q+3 times, and a sketch wider than one N-chunk is served by
// several CTAs per row tile, so the kernel above converts every entry of A (2q+3) x nch times —
// and the converters, not the tensor pipe, set its pace (ncu: tensor pipe 30 % active; F2I / PRMT
// streams on two to four warps per scheduler; the shared-memory pipe at ~75 % carrying the fp64
// staging next to the operands). Instead the decomposition converts A ONCE into its digit planes
// (k_oz_planes: one read of A, 14 bytes written per entry) and every A-pass is a pure int8 GEMM
// over them:
//   PN [7][rows][ldn]  slices of V = rint(a · 2^(54 - E_row)), K-major for op N (rows x cols)
//   PT [7][cols][ldt]  slices of rint(a · 2^(54 - F_col)), TRANSPOSED: K-major for op T (A^T is
//                      stored as digit planes; the fp64 A^T is still never formed)
// k_apass_ozp: warp 0 TMA producer (one 3-D box of the 7 A slices of the row tile + one of the 7
// X slices of the chunk per stage, SWIZZLE_32B), warp 1 MMA issuer (the same stacked MMAs),
// warps 4..7 read the level accumulators back at each flush. No converter, no fp64 staging: 139 KB
// of shared-memory traffic per stage instead of 203 KB, and A costs 7 B/entry/pass from HBM.
// (A slices through TMEM — tcgen05.st by the converters, "ts" MMAs — were measured too: 1.84 ms
// per C3 pass against 1.70 ms, the converters stay the bottleneck. TMA multicast of the A planes
// over a cluster of the row tile's chunk CTAs, with multicast commits on the empty barriers, was
// slower as well — C4 pass 8.5 vs 7.2 ms: four unicast reads of a line within a short window
// already cost L2 one read, and the cluster couples the four pipelines.)
constexpr int kPzStages = 5;
constexpr int kPzStage = kOzS * (kOzASlice + kOzXSlice);        // 42 KB
constexpr int kPzThreads = 256;
constexpr int kPzSmem = 1024 + kPzStages * kPzStage + 256;

__global__ void __launch_bounds__(kPzThreads, 1)
    k_apass_ozp(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmXa,
                const __grid_constant__ CUtensorMap tmXb, const __grid_constant__ OzArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kPzStages * kPzStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kPzStages;
    uint64_t* acc_full = empty + kPzStages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int bid = blockIdx.x;
    const int chunk = bid % p.nch;
    bid /= p.nch;
    const int mt = bid % p.mtiles;
    const int split = bid / p.mtiles;
    const int n0 = p.n0[chunk], nc = p.nc[chunk];
    const int64_t m0 = int64_t(mt) * kOzBM;
    const int64_t ktiles = (p.K + kOzBK - 1) / kOzBK;
    const int64_t kt0 = int64_t(split) * p.kt_per_split;
    const int nk = int((ktiles < kt0 + p.kt_per_split ? ktiles : kt0 + p.kt_per_split) - kt0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kPzStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmP)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(nc == p.nc_a ? &tmXa : &tmXb))
                     : "memory");
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
        // ===== TMA producer: the 7 A slices of the row tile and the 7 X slices of the chunk =====
        const uint32_t tx = uint32_t(kOzS * kOzASlice + kOzS * nc * kOzBK);
        for (int i = 0; i < nk; ++i) {
            const int s = i % kPzStages;
            const int k0 = int((kt0 + i) * kOzBK);
            if (i >= kPzStages) mbar_wait(&empty[s], ((i / kPzStages) - 1) & 1);
            if (lane == 0) {
                unsigned char* st = sm + s * kPzStage;
                mbar_expect_tx(&full[s], tx);
                tma_load_3d(st, &tmP, k0, int(m0), 0, &full[s]);
                tma_load_3d(st + kOzXOff, nc == p.nc_a ? &tmXa : &tmXb, k0, n0, 0, &full[s]);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        for (int i = 0; i < nk; ++i) {
            const int s = i % kPzStages;
            const int ci = i / kOzChunkStages;
            const bool first = (i % kOzChunkStages) == 0;
            if (first && ci > 0) mbar_wait(acc_empty, (ci - 1) & 1);
            mbar_wait(&full[s], (i / kPzStages) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t ab = smem_u32(sm + s * kPzStage);
                const uint32_t xb = ab + kOzXOff;
#pragma unroll
                for (int sl = 0; sl < kOzS; ++sl) {
                    // A slice sl x X slices 0..6-sl -> levels sl..6 (TMEM columns [sl·nc, 7·nc))
                    const int ntot = (kOzS - sl) * nc;
                    const uint64_t ad = sdesc_sw32(ab + sl * kOzASlice);
                    for (int c0 = 0; c0 < ntot; c0 += 256) {
                        const int n = ntot - c0 < 256 ? ntot - c0 : 256;
                        mma_i8(tmem + uint32_t(sl * nc + c0), ad, sdesc_sw32(xb + c0 * kOzBK), idesc_i8(n),
                               (first && sl == 0) ? 0u : 1u);
                    }
                }
                mma_commit(&empty[s]);
                if ((i % kOzChunkStages) == kOzChunkStages - 1 || i == nk - 1) mma_commit(acc_full);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== flushes: fp64 += sum_L acc_L 2^(-8L) · 2^(E + F_j - 12), own row, fixed order =====
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const int64_t row = m0 + r;
        const int E = row < p.Mo ? p.eA[row] : 0;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        double* out = p.split_stride > 0 ? p.C + split * p.split_stride + row * p.N : p.C + row * p.ldc;
        const int nfl = (nk + kOzChunkStages - 1) / kOzChunkStages;
        for (int f = 0; f < nfl; ++f) {
            mbar_wait(acc_full, f & 1);
            tc_fence_after();
            for (int cb = 0; cb < nc; cb += 8) {
                uint32_t acc[kOzS][8];
#pragma unroll
                for (int L = 0; L < kOzS; ++L) tmem_ld8(tmem + lane_base + uint32_t(L * nc + cb), acc[L]);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int col = n0 + cb + j;
                    double sum = double(int(acc[kOzS - 1][j]));
#pragma unroll
                    for (int L = kOzS - 2; L >= 0; --L) sum = fma(sum, 0.00390625, double(int(acc[L][j])));
                    if (row < p.Mo && col < p.N) {
                        const int ex = E + p.eX[col] - 12;
                        // sum · 2^ex in two exact steps (ex may leave the normal range of one factor)
                        const double val = (sum * pow2(ex >> 1)) * pow2(ex - (ex >> 1));
                        out[col] = f == 0 ? val : out[col] + val;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
    }
}

// A (rows x cols, lda) -> PN and PT. One 64 x 64 tile per CTA through shared memory (row stride 66
// doubles: the row-wise 16-byte reads of 8 consecutive rows and the column-wise 8-byte reads of 16
// consecutive columns are both conflict-free); a thread converts 16 entries of one row (row scale)
// and 16 entries of one column (column scale) and stores one 16-byte chunk per slice and plane.
constexpr int kPlTile = 64, kPlLd = 66;
__device__ __forceinline__ void oz_store_slices16(const double (&v)[16], double sc, uint8_t* dst, int64_t plane_stride) {
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const unsigned long long w = (unsigned long long)__double2ll_rn(v[j] * sc) + kOzBias;
        lo[j] = uint32_t(w);
        hi[j] = uint32_t(w >> 32);
    }
#pragma unroll
    for (int s = 0; s < kOzS; ++s) {
        const int b = 6 - s;
        uint32_t w4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t* src = b < 4 ? lo : hi;
            const uint32_t bb = uint32_t(b & 3);
            const uint32_t t01 = __byte_perm(src[4 * g], src[4 * g + 1], bb | ((bb + 4) << 4));
            const uint32_t t23 = __byte_perm(src[4 * g + 2], src[4 * g + 3], bb | ((bb + 4) << 4));
            w4[g] = __byte_perm(t01, t23, 0x5410) ^ (s == 0 ? 0u : 0x80808080u);
        }
        *reinterpret_cast<uint4*>(dst + s * plane_stride) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
}

__global__ void __launch_bounds__(256) k_oz_planes(const double* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                                   const int* __restrict__ erow, const int* __restrict__ ecol,
                                                   uint8_t* __restrict__ PN, int64_t ldn, uint8_t* __restrict__ PT,
                                                   int64_t ldt) {
    __shared__ __align__(16) double tile[kPlTile * kPlLd];
    const int64_t c0 = int64_t(blockIdx.x) * kPlTile, r0 = int64_t(blockIdx.y) * kPlTile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool vec = (lda & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        const int r = it * 8 + warp, c = 2 * lane;
        const int64_t gr = r0 + r, gc = c0 + c;
        double2 v = make_double2(0.0, 0.0);
        if (gr < rows) {
            if (vec && gc + 1 < cols) {
                v = *reinterpret_cast<const double2*>(A + gr * lda + gc);
            } else {
                if (gc < cols) v.x = A[gr * lda + gc];
                if (gc + 1 < cols) v.y = A[gr * lda + gc + 1];
            }
        }
        *reinterpret_cast<double2*>(&tile[r * kPlLd + c]) = v;
    }
    __syncthreads();
    {   // PN: row r = 8·warp + lane % 8, columns 16·(lane / 8) .. +15, row scale
        const int r = 8 * warp + (lane & 7), cq = lane >> 3;
        const int64_t gr = r0 + r, gc = c0 + 16 * cq;
        if (gr < rows && gc < cols) {
            double v[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double2 d2 = *reinterpret_cast<const double2*>(&tile[r * kPlLd + 16 * cq + 2 * i]);
                v[2 * i] = d2.x;
                v[2 * i + 1] = d2.y;
            }
            oz_store_slices16(v, pow2(54 - erow[gr]), PN + gr * ldn + gc, rows * ldn);
        }
    }
    {   // PT: column c = 16·(warp % 4) + lane % 16, rows 16·(2·(warp / 4) + lane / 16) .. +15, column scale
        const int c = 16 * (warp & 3) + (lane & 15), rg = 2 * (warp >> 2) + (lane >> 4);
        const int64_t gc = c0 + c, gr = r0 + 16 * rg;
        if (gc < cols && gr < rows) {
            double v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = tile[(16 * rg + j) * kPlLd + c];
            oz_store_slices16(v, pow2(54 - ecol[gc]), PT + gc * ldt + gr, cols * ldt);
        }
    }
}

// ---- exponents --------------------------------------------------------------------------------
__device__ __forceinline__ int biased_exp(double x) { return int((__double_as_longlong(x) >> 52) & 0x7ff); }

// Per-row and per-column maxima of the biased exponent field of A (rows x cols, lda): a CTA
// owns a 128-row x 512-column tile; thread = two adjacent columns (16-byte loads, 8 rows in
// flight), the row maxima go through warp reductions and shared memory, one integer atomicMax
// per row and per column per CTA — the result does not depend on the schedule.
constexpr int kExpRows = 128, kExpCols = 1024;
__global__ void __launch_bounds__(256) k_oz_aexp(const double* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                                 int* __restrict__ erow, int* __restrict__ ecol) {
    __shared__ int srow[kExpRows];
    const int64_t c = int64_t(blockIdx.x) * kExpCols + 4 * threadIdx.x;   // four consecutive columns per thread
    const int64_t r0 = int64_t(blockIdx.y) * kExpRows;
    for (int i = threadIdx.x; i < kExpRows; i += 256) srow[i] = 0;
    __syncthreads();
    const bool vec = (lda & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && c + 3 < cols;
    int cm[4] = {0, 0, 0, 0};
    for (int rr = 0; rr < kExpRows; rr += 4) {
        double x[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t r = r0 + rr + u;
#pragma unroll
            for (int q = 0; q < 4; ++q) x[u][q] = 0.0;
            if (r < rows) {
                if (vec) {
                    const double2 v0 = *reinterpret_cast<const double2*>(A + r * lda + c);
                    const double2 v1 = *reinterpret_cast<const double2*>(A + r * lda + c + 2);
                    x[u][0] = v0.x; x[u][1] = v0.y; x[u][2] = v1.x; x[u][3] = v1.y;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (c + q < cols) x[u][q] = A[r * lda + c + q];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int em = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int e = biased_exp(x[u][q]);
                e = e == 0x7ff ? 0x7fe : e;  // inf / nan: clamp (the host entry rejects them anyway)
                cm[q] = max(cm[q], e);
                em = max(em, e);
            }
            const int wm = int(__reduce_max_sync(0xffffffffu, unsigned(em)));
            if ((threadIdx.x & 31) == 0 && wm > 0) atomicMax(&srow[rr + u], wm);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (c + q < cols && cm[q] > 0) atomicMax(&ecol[c + q], cm[q]);
    __syncthreads();
    for (int i = threadIdx.x; i < kExpRows; i += 256)
        if (r0 + i < rows && srow[i] > 0) atomicMax(&erow[r0 + i], srow[i]);
}

__global__ void k_oz_finish_exp(int* __restrict__ e, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        e[i] = oz_exp_from_biased(e[i]);
}

// Per-column maxima of the biased exponent of X (K x N, ldx).
__global__ void __launch_bounds__(256) k_oz_xexp(const double* __restrict__ X, int64_t ldx, int64_t K, int N,
                                                 int* __restrict__ fmax) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + tx;
    int m = 0;
    for (int64_t k = int64_t(blockIdx.y) * 8 + ty; k < K; k += int64_t(gridDim.y) * 8)
        if (c < N) m = max(m, biased_exp(X[k * ldx + c]));
    if (c < N) atomicMax(&fmax[c], m == 0x7ff ? 0x7fe : m);
}

// X (K x N) -> 7 balanced digit slices, K-major: Xs[(s·xrows + n)·ldk + k] = digit s of W_kn,
// W = rint(x · 2^(54 - F_n)); zero for n >= N and k >= K. 128(k) x 32(n) tiles through shared
// memory, stored transposed (k contiguous): a thread converts 4 consecutive k of one column and
// stores one 32-bit word per slice, a warp 128 contiguous bytes of one slice row (the 32-k tiles
// of the first version wrote 32-byte pieces: 90 us for C3's 200000 x 110 c1).
constexpr int kSplitK = 128, kSplitLd = kSplitK + 2;
__global__ void __launch_bounds__(256) k_oz_split_x(const double* __restrict__ X, int64_t ldx, int64_t K, int N,
                                                    const int* __restrict__ fexp, int xrows, int64_t ldk,
                                                    uint8_t* __restrict__ Xs) {
    __shared__ __align__(16) double tile[32 * kSplitLd];
    const int64_t k0 = int64_t(blockIdx.x) * kSplitK;
    const int nb = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll 4
    for (int rr = ty; rr < kSplitK; rr += 8) {
        const int64_t k = k0 + rr;
        const int n = nb + tx;
        tile[tx * kSplitLd + rr] = (k < K && n < N) ? X[k * ldx + n] : 0.0;
    }
    __syncthreads();
    const int kg = tx;  // 4 consecutive k: 4·kg ..
    const int64_t k = k0 + 4 * kg;
    for (int nn = ty; nn < 32; nn += 8) {
        const int n = nb + nn;
        if (n >= xrows || k >= ldk) continue;
        const double sc = n < N ? pow2(54 - fexp[n]) : 0.0;
        const double2 v01 = *reinterpret_cast<const double2*>(&tile[nn * kSplitLd + 4 * kg]);
        const double2 v23 = *reinterpret_cast<const double2*>(&tile[nn * kSplitLd + 4 * kg + 2]);
        const double v[4] = {v01.x, v01.y, v23.x, v23.y};
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned long long w = (unsigned long long)__double2ll_rn(v[j] * sc) + kOzBias;
            lo[j] = uint32_t(w);
            hi[j] = uint32_t(w >> 32);
        }
#pragma unroll
        for (int s2 = 0; s2 < kOzS; ++s2) {
            const int bq = 6 - s2;
            const uint32_t* src = bq < 4 ? lo : hi;
            const uint32_t bb = uint32_t(bq & 3);
            const uint32_t t01 = __byte_perm(src[0], src[1], bb | ((bb + 4) << 4));
            const uint32_t t23 = __byte_perm(src[2], src[3], bb | ((bb + 4) << 4));
            *reinterpret_cast<uint32_t*>(Xs + (int64_t(s2) * xrows + n) * ldk + k) =
                __byte_perm(t01, t23, 0x5410) ^ (s2 == 0 ? 0u : 0x80808080u);
        }
    }
}

__global__ void k_oz_finish_xexp(int* __restrict__ f, int N) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) f[i] = oz_exp_from_biased(f[i]);
}

__global__ void k_oz_reduce(const double* __restrict__ P, int64_t split_stride, int splits, double* __restrict__ C,
                            int64_t ldc, int64_t rows, int N) {
    const int64_t total = rows * N;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        double s = P[e];
        for (int k = 1; k < splits; ++k) s += P[k * split_stride + e];
        C[(e / N) * ldc + e % N] = s;
    }
}

// ---- host side ----------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() {
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

bool oz_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, const cuuint64_t* dims, cuuint64_t stride_bytes,
            const cuuint32_t* box, CUtensorMapSwizzle sw) {
    auto fn = oz_encode_fn();
    if (!fn) return false;
    const cuuint64_t str[1] = {stride_bytes};
    const cuuint32_t es[2] = {1, 1};
    return fn(m, dt, 2, const_cast<void*>(base), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct OzShape {
    int nch, n0[kOzMaxChunks], nc[kOzMaxChunks], xrows;
    int mtiles, splits, kt_per_split;
    int64_t ldk;
};

OzShape oz_shape(int64_t Mo, int64_t K, int N, int num_sms) {
    OzShape s{};
    const int n16 = (N + 15) / 16 * 16;
    s.nch = (n16 + kOzNcMax - 1) / kOzNcMax;
    const int units = n16 / 16;  // 16-column units spread over the chunks, larger chunks first
    int at = 0;
    for (int c = 0; c < s.nch; ++c) {
        const int u = units / s.nch + (c < units % s.nch ? 1 : 0);
        s.n0[c] = at;
        s.nc[c] = 16 * u;
        at += 16 * u;
    }
    s.xrows = n16;
    s.ldk = (K + 15) / 16 * 16;
    s.mtiles = int((Mo + kOzBM - 1) / kOzBM);
    const int64_t ktiles = (K + kOzBK - 1) / kOzBK;
    const int64_t base = int64_t(s.mtiles) * s.nch;
    double best = 1e30;
    int best_s = 1;
    const int max_s = int(std::max<int64_t>(1, std::min<int64_t>(ktiles / 64, 32)));
    for (int sp = 1; sp <= max_s; ++sp) {
        const double waves = std::ceil(double(base * sp) / num_sms);
        const double cost = waves / sp + (sp > 1 ? 0.02 : 0.0);
        if (cost < best - 1e-12) {
            best = cost;
            best_s = sp;
        }
    }
    s.kt_per_split = int((ktiles + best_s - 1) / best_s);
    s.splits = int((ktiles + s.kt_per_split - 1) / s.kt_per_split);
    return s;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

bool gemm_oz_eligible(int64_t Mo, int64_t K, int N) {
    return N >= 1 && N <= kOzMaxChunks * kOzNcMax && Mo >= kOzBM && K >= 8 * kOzBK && K < (int64_t(1) << 31) &&
           Mo < (int64_t(1) << 31);
}

bool gemm_oz_supported(Op op, const double* A, int64_t lda, int64_t Mo, int64_t K, int N) {
    (void)op;
    if (!oz_encode_fn() || !gemm_oz_eligible(Mo, K, N)) return false;
    return (lda * 8) % 16 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
}

size_t gemm_oz_ws_bytes(int64_t Mo, int64_t K, int N, int num_sms) {
    const OzShape s = oz_shape(Mo, K, N, num_sms);
    size_t b = align_up(size_t(kOzS) * s.xrows * size_t(s.ldk), 256);  // X slices
    b += align_up(sizeof(int) * size_t(N), 256);                        // X exponents
    if (s.splits > 1) b += sizeof(double) * size_t(s.splits) * size_t(Mo) * size_t(N);
    return b + 256;
}

cudaError_t gemm_oz_exponents_begin(int64_t rows, int64_t cols, int* erow, int* ecol, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(erow, 0, sizeof(int) * size_t(rows), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ecol, 0, sizeof(int) * size_t(cols), st);
    return e;
}
cudaError_t gemm_oz_exponents_rows(const double* A, int64_t lda, int64_t r0, int64_t nrows, int64_t cols, int* erow,
                                   int* ecol, cudaStream_t st) {
    const dim3 grid(unsigned((cols + kExpCols - 1) / kExpCols), unsigned((nrows + kExpRows - 1) / kExpRows));
    k_oz_aexp<<<grid, 256, 0, st>>>(A + r0 * lda, lda, nrows, cols, erow + r0, ecol);
    return cudaGetLastError();
}
cudaError_t gemm_oz_exponents_end(int64_t rows, int64_t cols, int* erow, int* ecol, cudaStream_t st) {
    k_oz_finish_exp<<<int(std::min<int64_t>((rows + 255) / 256, 1184)), 256, 0, st>>>(erow, rows);
    k_oz_finish_exp<<<int(std::min<int64_t>((cols + 255) / 256, 1184)), 256, 0, st>>>(ecol, cols);
    return cudaGetLastError();
}
cudaError_t gemm_oz_exponents(const double* A, int64_t lda, int64_t rows, int64_t cols, int* erow, int* ecol,
                              cudaStream_t st) {
    cudaError_t e = gemm_oz_exponents_begin(rows, cols, erow, ecol, st);
    if (e == cudaSuccess) e = gemm_oz_exponents_rows(A, lda, 0, rows, cols, erow, ecol, st);
    if (e == cudaSuccess) e = gemm_oz_exponents_end(rows, cols, erow, ecol, st);
    return e;
}

OzPlaneDims gemm_oz_plane_dims(int64_t rows, int64_t cols) {
    OzPlaneDims d;
    // plane rows start on 128-byte lines: a 32-byte box row never straddles two L2 sectors (an
    // unaligned row pitch cost 1.5x the L2 -> SM traffic: ncu l1tex__m_xbar2l1tex_read_bytes)
    d.ldn = (cols + 127) / 128 * 128;
    d.ldt = (rows + 127) / 128 * 128;
    d.pn_bytes = align_up(size_t(kOzS) * size_t(rows) * size_t(d.ldn), 256);
    d.pt_bytes = align_up(size_t(kOzS) * size_t(cols) * size_t(d.ldt), 256);
    return d;
}

cudaError_t gemm_oz_planes(const double* A, int64_t lda, int64_t rows, int64_t cols, const int* erow, const int* ecol,
                           uint8_t* planes, cudaStream_t st) {
    const OzPlaneDims d = gemm_oz_plane_dims(rows, cols);
    const dim3 grid(unsigned((cols + kPlTile - 1) / kPlTile), unsigned((rows + kPlTile - 1) / kPlTile));
    k_oz_planes<<<grid, 256, 0, st>>>(A, lda, rows, cols, erow, ecol, planes, d.ldn, planes + d.pn_bytes, d.ldt);
    return cudaGetLastError();
}

cudaError_t gemm_oz(Op op, const double* A, int64_t lda, const OzPlanes* pl, const int* eA, const double* X,
                    int64_t ldx, double* C, int64_t ldc, int64_t Mo, int64_t K, int N, void* ws, int num_sms,
                    cudaStream_t st, const OzPlanes* store) {
    if (store && (pl || op != Op::N)) return cudaErrorInvalidValue;
    const OzShape s = oz_shape(Mo, K, N, num_sms);
    unsigned char* w = static_cast<unsigned char*>(ws);
    uint8_t* xs = w;
    w += align_up(size_t(kOzS) * s.xrows * size_t(s.ldk), 256);
    int* fx = reinterpret_cast<int*>(w);
    w += align_up(sizeof(int) * size_t(N), 256);
    double* part = reinterpret_cast<double*>(w);
    cudaError_t e = cudaMemsetAsync(fx, 0, sizeof(int) * size_t(N), st);
    if (e != cudaSuccess) return e;
    {
        const int gy = int(std::max<int64_t>(1, std::min<int64_t>((K + 7) / 8, 1184 / ((N + 31) / 32) + 1)));
        k_oz_xexp<<<dim3(unsigned((N + 31) / 32), unsigned(gy)), 256, 0, st>>>(X, ldx, K, N, fx);
        k_oz_finish_xexp<<<(N + 255) / 256, 256, 0, st>>>(fx, N);
        const dim3 grid(unsigned((s.ldk + kSplitK - 1) / kSplitK), unsigned((s.xrows + 31) / 32));
        k_oz_split_x<<<grid, 256, 0, st>>>(X, ldx, K, N, fx, s.xrows, s.ldk, xs);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    CUtensorMap ta, tx, tp;
    // digit planes of op(A): (k, row, slice), one box = the 7 slices of a 128-row tile
    auto pmap = [&](CUtensorMap* m, const OzPlanes* q) {
        auto fn = oz_encode_fn();
        const cuuint64_t dims[3] = {cuuint64_t(K), cuuint64_t(Mo), cuuint64_t(kOzS)};
        const cuuint64_t str[2] = {cuuint64_t(q->ld), cuuint64_t(q->ld) * cuuint64_t(q->rows)};
        const cuuint32_t box[3] = {kOzBK, kOzBM, cuuint32_t(kOzS)};
        const cuuint32_t es[3] = {1, 1, 1};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(q->p), dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (store && !pmap(&tp, store)) return cudaErrorInvalidValue;
    if (pl) {
        if (!pmap(&ta, pl)) return cudaErrorInvalidValue;
    } else if (op == Op::N) {
        const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(Mo)};
        const cuuint32_t box[2] = {16, kOzBM};
        if (!oz_map(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, A, dims, cuuint64_t(lda) * 8, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    } else {
        const cuuint64_t dims[2] = {cuuint64_t(Mo), cuuint64_t(K)};
        const cuuint32_t box[2] = {kOzBM, kOzBK};
        if (!oz_map(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, A, dims, cuuint64_t(lda) * 8, box, CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    }
    // X slices as a 3-D tensor (k, row, slice); one box = the 7 slices of one chunk, stacked.
    auto xmap = [&](CUtensorMap* m, int nc) {
        auto fn = oz_encode_fn();
        const cuuint64_t dims[3] = {cuuint64_t(K), cuuint64_t(s.xrows), cuuint64_t(kOzS)};
        const cuuint64_t str[2] = {cuuint64_t(s.ldk), cuuint64_t(s.ldk) * cuuint64_t(s.xrows)};
        const cuuint32_t box[3] = {kOzBK, cuuint32_t(nc), cuuint32_t(kOzS)};
        const cuuint32_t es[3] = {1, 1, 1};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, xs, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    CUtensorMap txb;
    const int nc_a = s.nc[0], nc_b = s.nc[s.nch - 1];
    if (!xmap(&tx, nc_a) || !xmap(&txb, nc_b)) return cudaErrorInvalidValue;
    OzArgs a{};
    a.Mo = Mo;
    a.K = K;
    a.N = N;
    a.nch = s.nch;
    for (int c = 0; c < kOzMaxChunks; ++c) {
        a.n0[c] = s.n0[c];
        a.nc[c] = s.nc[c];
    }
    a.xrows = s.xrows;
    a.nc_a = nc_a;
    a.mtiles = s.mtiles;
    a.kt_per_split = s.kt_per_split;
    a.C = s.splits > 1 ? part : C;
    a.ldc = ldc;
    a.split_stride = s.splits > 1 ? Mo * N : 0;
    a.eA = eA;
    a.eX = fx;
    const unsigned grid = unsigned(int64_t(s.nch) * s.mtiles * s.splits);
    if (pl) {
        allow_max_smem(k_apass_ozp);
        k_apass_ozp<<<grid, kPzThreads, kPzSmem, st>>>(ta, tx, txb, a);
    } else if (op == Op::N && store) {
        allow_max_smem(k_apass_oz<false, true>);
        k_apass_oz<false, true><<<grid, kOzThreads, kOzSmem, st>>>(ta, tx, txb, tp, a);
    } else if (op == Op::N) {
        allow_max_smem(k_apass_oz<false, false>);
        k_apass_oz<false, false><<<grid, kOzThreads, kOzSmem, st>>>(ta, tx, txb, ta, a);
    } else {
        allow_max_smem(k_apass_oz<true, false>);
        k_apass_oz<true, false><<<grid, kOzThreads, kOzSmem, st>>>(ta, tx, txb, ta, a);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess || s.splits == 1) return e;
    const int64_t total = Mo * N;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(num_sms) * 8));
    k_oz_reduce<<<blocks, 256, 0, st>>>(part, Mo * N, s.splits, C, ldc, Mo, N);
    return cudaGetLastError();
}

int gemm_oz_launches(int64_t Mo, int64_t K, int N, int num_sms) {
    return 4 + (oz_shape(Mo, K, N, num_sms).splits > 1 ? 1 : 0);
}

}  // namespace coru_gpu
