// C-ABI (include/coru_gpu.h) and host orchestration of CoR-UTV on B200.
//
// The step order is the reference's (corutv.hpp:49-100):
//   Φ = gaussian(n, ell, seed)                        host, bit-exact (rng_host.cpp), one H2D
//   q+1 x { B1 = A·B2 ; B2 = A^T·B1 }                  gemm (op N / op T: A^T is never formed)
//   Q1,R1 = TSQR(B1) ; Q2 = TSQR(B2)                    tsqr.cu (R-tree, explicit Q)
//   warning = |R1(ell,ell)| <= 1e-14 |R1(1,1)|
//   D = Q1^T (A Q2)                                     two gemm calls; W = A·Q2 is m x ell
//   Q_M, T, perm = QRCP(D) ; U = Q1·Q_M ; V = Q2·P       qrcp.cu + gemm + gather
// With a communicator (A row-sharded over ranks) the A^T-products and D are summed with
// ncclAllReduce, the B1 TSQR tree gets a cross-rank top level (ncclAllGather of the ell x ell R's,
// redundant top QR on every rank), and everything ell x ell or n x ell is computed redundantly
// and bit-identically on every rank (all kernels are atomic-free and fixed-order).
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cstdlib>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <emmintrin.h>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/coru_gpu.h"
#include "gemm.cuh"
#include "qrcp.cuh"
#include "cholqr.cuh"
#include "rng_dev.cuh"
#include "rpca.cuh"
#include "svd.cuh"
#include "tsqr.cuh"

namespace coru_gpu {
void host_parallel(int n, const std::function<void(int)>& f);
template <typename OutT>
void gaussian_host(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, OutT* out, int64_t ldo, int threads,
                   int streaming);
template <typename OutT>
void gaussian_host_rows(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, OutT* out, int64_t ldo,
                        int threads, int streaming, int64_t r0, int64_t r1);
}  // namespace coru_gpu

using namespace coru_gpu;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CORU_CUDA(expr)                                                                                      \
    do {                                                                                                     \
        cudaError_t e_ = (expr);                                                                             \
        if (e_ != cudaSuccess) return fail(CORU_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));  \
    } while (0)

#define CORU_TRY(expr)                  \
    do {                                \
        int rc_ = (expr);               \
        if (rc_ != CORU_OK) return rc_; \
    } while (0)

// ---- NCCL, loaded at run time ------------------------------------------------------------------
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string err;
};

Nccl* nccl() {
    static Nccl api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* nm : {"libnccl.so.2", "libnccl.so"})
            if ((api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!api.h) {
            api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
#define LOAD(sym) api.sym = reinterpret_cast<decltype(api.sym)>(dlsym(api.h, "nccl" #sym))
        LOAD(GetUniqueId);
        LOAD(CommInitRank);
        LOAD(CommDestroy);
        LOAD(AllReduce);
        LOAD(AllGather);
        LOAD(GetErrorString);
#undef LOAD
        if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather || !api.GetErrorString) {
            api.err = "libnccl is missing required symbols";
            api.h = nullptr;
        }
    });
    return api.h ? &api : nullptr;
}

#define CORU_NCCL(expr)                                                                               \
    do {                                                                                              \
        ncclResult_t r_ = (expr);                                                                     \
        if (r_ != ncclSuccess) return fail(CORU_ENCCL, std::string(#expr) + ": " + nccl()->GetErrorString(r_)); \
    } while (0)

template <typename T>
ncclDataType_t nccl_type() {
    return sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
constexpr int kTnMaxBlocks = 592;  // row blocks of the skinny Q^T·W kernel (tn_small)

// Bump allocator: a measuring pass (base == nullptr) then a carving pass over the arena.
struct Carver {
    char* base = nullptr;
    size_t off = 0;
    template <typename T>
    T* take(int64_t n) {
        off = (off + 255) / 256 * 256;
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += size_t(std::max<int64_t>(n, 0)) * sizeof(T);
        return p;
    }
};

}  // namespace

// In-process collective group: ranks are host threads (each with its own context, on one GPU or
// on peer-accessible GPUs). A collective = stream sync + host barrier + fixed-order device sum /
// copies, so it is deterministic and no kernel ever waits on another kernel.
struct coru_threadcomm {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<const void*> slots;
    std::vector<int> devices;  // device of each rank (-1: not joined yet)
    bool failed = false;  // a rank failed: every pending and future barrier returns false
    explicit coru_threadcomm(int w) : world(w), slots(size_t(w), nullptr), devices(size_t(w), -1) {}
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (failed) return false;
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen || failed; });
        }
        return !failed;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        failed = true;
        cv.notify_all();
    }
};

struct coru_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // second stream: the two TSQR trees run concurrently
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_phi = nullptr;  // last H2D copy out of the pinned Φ staging buffer
    // Φ of the NEXT inner decomposition of an iterative caller (alm_rpca: substream(seed, it + 1)),
    // generated by a background host thread into its own pinned buffer while the GPU finishes the
    // current iteration.
    // CUDA-graph replay of small decompositions (launch-bound: C1, C2): one instantiated graph per
    // (A, shape, parameters, output buffers), captured on the second call with the same key.
    struct GraphEntry {
        const void *A = nullptr, *u = nullptr, *t = nullptr, *v = nullptr, *arena = nullptr, *pinned = nullptr;
        int64_t lda = 0, rows = 0, cols = 0, ldu = 0, ldt = 0, ldv = 0;
        int d = 0, q = 0, variant = 0, elem = 0;
        bool trans = false, want_perm = false;
        cudaStream_t stream = nullptr;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        int state = 0;  // 0 seen once, 1 instantiated, -1 capture failed (never again)
        uint64_t last_use = 0;
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_clock = 0;
    int64_t graph_replays = 0;
    int64_t* host_out = nullptr;  // pinned: [0] conditioning flag, [1..] pivots (graph replays write here)
    std::thread pf_thread;
    bool pf_active = false;
    uint64_t pf_seed = 0, pf_stream = 0;
    int64_t pf_rows = 0;
    int pf_cols = 0, pf_ld = 0;
    size_t pf_elem = 0;
    char* pf_buf = nullptr;
    size_t pf_bytes = 0;
    cudaEvent_t ev_pf = nullptr;
    static constexpr int kUploadChunks = 8;
    cudaEvent_t ev_chunk[kUploadChunks] = {};  // host-entry upload pipeline (corutv_host)
    int num_sms = 148;
    int max_smem = 227 * 1024;
    int host_threads = 1;
    int phi_mode = CORU_PHI_HOST_EXACT;  // the reference's Φ bit for bit (rng.hpp:86-112)
    int f32_path = CORU_F32_AUTO;
    int f64_engine = CORU_F64_AUTO;
    // Ozaki A-pass state (gemm_oz.cu): the exponents of the matrix the current call streams
    // (prepared at the start of a decomposition, cleared at its end — never reused across calls).
    const double* oz_a = nullptr;
    int64_t oz_lda = 0, oz_rows = 0, oz_cols = 0;
    int* oz_e = nullptr;        // erow [oz_rows] then ecol [oz_cols]
    size_t oz_e_cap = 0;        // ints
    void* oz_ws = nullptr;
    size_t oz_ws_bytes = 0;
    // Digit planes of the prepared matrix (converted once per decomposition; gemm_oz.cu). Null when
    // they do not fit next to A (then the A-pass kernel converts A itself on every pass).
    void* oz_planes = nullptr;
    size_t oz_planes_cap = 0;
    bool oz_planes_ready = false;
    int oz_pn_state = 0;        // hybrid: 0 off, 1 the next full op-N pass writes the PN planes, 2 PN planes valid
    // exponents already in oz_e for this matrix (the host entry computes them chunk by chunk under the upload)
    const double* oz_pre_a = nullptr;
    int64_t oz_pre_lda = 0, oz_pre_rows = 0, oz_pre_cols = 0;
    int last_f64_engine = 0;  // engine of the last fp64 A-pass: 0 DMMA, 1 Ozaki (in-kernel digits), 2 Ozaki (digit planes), 3 Ozaki hybrid
    bool wide_qr = true;  // CholeskyQR2 (fp64) for sketches wider than 128 columns, Householder fall-back
    char* arena = nullptr;
    size_t arena_bytes = 0;
    char* pinned = nullptr;
    size_t pinned_bytes = 0;
    // Staging ring for pageable host buffers (std::vector / coru::Matrix storage): the host worker
    // pool copies piece k+1 into a pinned slot while the DMA engine moves piece k.
    static constexpr int kStageSlots = 4;
    static constexpr size_t kStageBytes = size_t(16) << 20;
    bool stage_nt = false;  // streaming (non-temporal) stores into the ring: CORU_STAGE_NT=1 (tooling)
    char* stage = nullptr;
    cudaEvent_t ev_stage[kStageSlots] = {};
    int stage_next = 0;
    ncclComm_t comm = nullptr;
    coru_threadcomm* tcomm = nullptr;  // in-process backend (instead of NCCL)
    void* tscratch = nullptr;          // its reduction scratch
    size_t tscratch_bytes = 0;
    int rank = 0, world = 1;
    std::mutex mu;
    // A-pass profiling (bench evidence): CUDA events recorded on the launching stream around every
    // GEMM that streams the caller's A, plus their algorithmic flop and byte counts.
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;
    double prof_flops = 0, prof_bytes = 0;
    // A-passes issued while another stream of the same call runs QR kernels (early Q1 tree, late
    // join) share the SMs with them: flagged, so the roofline can also be read from the passes that
    // had the GPU to themselves.
    bool prof_overlap = false;
    std::vector<char> prof_shared;
    // the same for the fused ALM lift + update kernel of alm_rpca (rpca.cu)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> upd_events;
    size_t upd_used = 0;
    double upd_flops = 0, upd_bytes = 0;
};

namespace {

int ensure_arena(coru_ctx* c, size_t bytes) {
    if (bytes <= c->arena_bytes) return CORU_OK;
    if (c->arena) {
        CORU_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(c->arena);
        c->arena = nullptr;
        c->arena_bytes = 0;
    }
    const size_t want = bytes + bytes / 8 + (1 << 20);
    if (cudaMalloc(&c->arena, want) != cudaSuccess) {
        cudaGetLastError();
        return fail(CORU_ENOMEM, "cudaMalloc of " + std::to_string(want) + " workspace bytes failed");
    }
    c->arena_bytes = want;
    return CORU_OK;
}

int ensure_pinned(coru_ctx* c, size_t bytes) {
    if (bytes <= c->pinned_bytes) return CORU_OK;
    if (c->pinned) {
        CORU_CUDA(cudaStreamSynchronize(c->stream));
        cudaFreeHost(c->pinned);
        c->pinned = nullptr;
        c->pinned_bytes = 0;
    }
    if (cudaMallocHost(&c->pinned, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(CORU_ENOMEM, "cudaMallocHost of " + std::to_string(bytes) + " bytes failed");
    }
    c->pinned_bytes = bytes;
    return CORU_OK;
}

bool is_pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int ensure_stage(coru_ctx* c) {
    if (c->stage) return CORU_OK;
    if (cudaMallocHost(&c->stage, coru_ctx::kStageBytes * coru_ctx::kStageSlots) != cudaSuccess) {
        cudaGetLastError();
        c->stage = nullptr;
        return fail(CORU_ENOMEM, "cudaMallocHost of the staging ring failed");
    }
    for (auto& e : c->ev_stage) CORU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return CORU_OK;
}

// Copy with streaming stores (no read-for-ownership of the destination, no cache pollution): for
// destinations the CPU will not read again — the pinned ring the DMA engine drains.
void memcpy_stream(char* dst, const char* src, size_t n) {
    while (n && (reinterpret_cast<uintptr_t>(dst) & 15)) {
        *dst++ = *src++;
        --n;
    }
    size_t i = 0;
    for (; i + 64 <= n; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
        const __m128i c2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
        const __m128i d2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c2);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d2);
    }
    if (i < n) std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}

// memcpy on the host worker pool (pieces of >= 1 MB per worker).
void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads, bool stream_stores = false) {
    const int nt = int(std::max<size_t>(1, std::min<size_t>(size_t(std::max(threads, 1)), bytes >> 20)));
    host_parallel(nt, [&](int t) {
        const size_t b0 = bytes * size_t(t) / size_t(nt), b1 = bytes * size_t(t + 1) / size_t(nt);
        if (stream_stores)
            memcpy_stream(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, b1 - b0);
        else
            std::memcpy(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, b1 - b0);
    });
}

// Piece size of the staging ring: 8 MB, one worker per MB — measured best on the 16-core host (C3
// pageable e2e 13.0 decompositions/s; 16 MB x 16 workers 12.5, 4 MB 7.6, streaming stores 11.6 — the
// ring then no longer stays in the CPU caches the DMA engine reads it from). CORU_STAGE_MB: tooling.
size_t stage_piece_bytes() {
    static const size_t piece = [] {
        const char* e = getenv("CORU_STAGE_MB");
        const size_t mb = e ? size_t(std::max(1, std::min(16, atoi(e)))) : 8;
        return mb << 20;
    }();
    return piece;
}

// Host -> device copy of `bytes` on `st`. Page-locked sources go straight to the DMA engine; pageable
// ones (the drop-in caller's std::vector storage) are staged through the pinned ring: the host pool
// fills slot k+1 while the DMA engine drains slot k, so the copy runs near link speed instead of the
// driver's synchronous pageable path. Returns once every piece is enqueued.
int h2d(coru_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return CORU_OK;
    if (is_pinned_host(src)) {
        CORU_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return CORU_OK;
    }
    CORU_TRY(ensure_stage(c));
    const size_t piece = stage_piece_bytes();
    for (size_t off = 0; off < bytes; off += piece) {
        const size_t len = std::min(piece, bytes - off);
        const int b = c->stage_next;
        c->stage_next = (b + 1) % coru_ctx::kStageSlots;
        char* slot = c->stage + size_t(b) * coru_ctx::kStageBytes;
        CORU_CUDA(cudaEventSynchronize(c->ev_stage[b]));  // the slot's previous DMA has drained
        parallel_memcpy(slot, static_cast<const char*>(src) + off, len, c->host_threads, c->stage_nt);
        CORU_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, slot, len, cudaMemcpyHostToDevice, st));
        CORU_CUDA(cudaEventRecord(c->ev_stage[b], st));
    }
    return CORU_OK;
}

// Device -> host copy; synchronises `st`. Pageable destinations: piece k+1 is in flight while the
// host pool copies piece k out of its slot.
int d2h_sync(coru_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return CORU_OK;
    if (is_pinned_host(dst)) {
        CORU_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaStreamSynchronize(st));
        return CORU_OK;
    }
    CORU_TRY(ensure_stage(c));
    static const size_t Pd = [] {  // CORU_STAGE_D2H_MB: tooling (slot stride stays kStageBytes)
        const char* e = getenv("CORU_STAGE_D2H_MB");
        return size_t(e ? std::max(1, std::min(16, atoi(e))) : 16) << 20;
    }();
    const size_t P = Pd;
    const size_t pieces = (bytes + P - 1) / P;
    auto issue = [&](size_t k) -> int {
        const int b = int(k % coru_ctx::kStageSlots);
        const size_t off = k * P, len = std::min(P, bytes - off);
        CORU_CUDA(cudaMemcpyAsync(c->stage + size_t(b) * coru_ctx::kStageBytes, static_cast<const char*>(src) + off, len,
                                  cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaEventRecord(c->ev_stage[b], st));
        return CORU_OK;
    };
    const size_t ahead = coru_ctx::kStageSlots - 1;
    for (size_t k = 0; k < std::min(pieces, ahead); ++k) CORU_TRY(issue(k));
    for (size_t k = 0; k < pieces; ++k) {
        const int b = int(k % coru_ctx::kStageSlots);
        const size_t off = k * P, len = std::min(P, bytes - off);
        CORU_CUDA(cudaEventSynchronize(c->ev_stage[b]));
        parallel_memcpy(static_cast<char*>(dst) + off, c->stage + size_t(b) * coru_ctx::kStageBytes, len, c->host_threads);
        if (k + ahead < pieces) CORU_TRY(issue(k + ahead));
    }
    return CORU_OK;
}

// Grow-only device buffer owned by the context (synchronises its stream before a regrow).
int ensure_dev(coru_ctx* c, void** buf, size_t* cap, size_t bytes, const char* what) {
    if (bytes <= *cap) return CORU_OK;
    if (*buf) {
        CORU_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(*buf);
        *buf = nullptr;
        *cap = 0;
    }
    if (cudaMalloc(buf, bytes) != cudaSuccess) {
        cudaGetLastError();
        *buf = nullptr;
        return fail(CORU_ENOMEM, std::string("cudaMalloc of ") + std::to_string(bytes) + " bytes (" + what + ") failed");
    }
    *cap = bytes;
    return CORU_OK;
}

bool oz_enabled(const coru_ctx* c) {
    static const char* env = getenv("CORU_F64_ENGINE");  // tooling override: dmma | ozaki
    if (env && std::string(env) == "dmma") return false;
    if (env && std::string(env) == "ozaki") return true;
    return c->f64_engine != CORU_F64_DMMA;
}

// Exponents of the stored matrix (rows x cols, lda) the coming A-passes stream (gemm_oz.cu): one
// extra read of A per decomposition, reused by every pass over it.
// passes: A-passes the caller will run over A; ncols: their sketch width (decides digit planes).
// passes_n: how many of them are op-N passes over the stored matrix (decides the hybrid mode).
// Will the A-passes over a rows x cols matrix with an ncols-wide sketch run on the Ozaki engine?
bool oz_wanted(const coru_ctx* c, int64_t rows, int64_t cols, int ncols) {
    if (!oz_enabled(c)) return false;
    if (!gemm_oz_eligible(std::max(rows, cols), std::min(rows, cols), 1)) return false;
    // The int8 kernel runs one CTA per (128-row tile, 64-column chunk): on a small matrix it cannot
    // fill the machine and the FP64 stream-K kernel is faster (C2, 4000^2 x 60: 32 CTAs, 187 us per
    // pass against 83 us on DMMA; C1 likewise). Forced engines skip the test.
    if (c->f64_engine == CORU_F64_AUTO && getenv("CORU_F64_ENGINE") == nullptr) {
        const int64_t ctas = ((std::max(rows, cols) + 127) / 128) * ((ncols + 63) / 64);
        if (ctas < 2 * int64_t(c->num_sms)) return false;  // under two waves: DMMA (RPCA 8000^2 x 80 too)
    }
    return true;
}
int oz_ensure_exponents(coru_ctx* c, int64_t rows, int64_t cols) {
    size_t cap_bytes = c->oz_e_cap * sizeof(int);
    void* e = c->oz_e;
    CORU_TRY(ensure_dev(c, &e, &cap_bytes, sizeof(int) * size_t(rows + cols), "Ozaki exponents"));
    c->oz_e = static_cast<int*>(e);
    c->oz_e_cap = cap_bytes / sizeof(int);
    return CORU_OK;
}

int oz_prepare(coru_ctx* c, const double* A, int64_t lda, int64_t rows, int64_t cols, int passes, int ncols,
               int passes_n = 0) {
    c->oz_a = nullptr;
    c->last_f64_engine = 0;
    c->oz_pn_state = 0;
    const bool pre = A && c->oz_pre_a == A && c->oz_pre_lda == lda && c->oz_pre_rows == rows && c->oz_pre_cols == cols;
    c->oz_pre_a = nullptr;
    if (!A || !oz_wanted(c, rows, cols, ncols)) return CORU_OK;
    if (!pre) {
        CORU_TRY(oz_ensure_exponents(c, rows, cols));
        CORU_CUDA(gemm_oz_exponents(A, lda, rows, cols, c->oz_e, c->oz_e + rows, c->stream));
        g_launches += 3;
    }
    // Digit planes (14 bytes per entry): converted once here, streamed by every A-pass. Skipped when
    // they would not fit in what is free now (beyond what the context already holds for them).
    // Worth it when the conversion would otherwise be repeated often enough: every pass converts A
    // once per 64-column chunk of the sketch inside the A-pass kernel. Measured on B200: C3 (5
    // passes x 2 chunks) 17.0 ms inline vs 18.2 ms with planes, C4 (7 x 4) 87.0 vs 83.5 ms.
    c->oz_planes_ready = false;
    static const char* planes_env = getenv("CORU_OZ_PLANES");  // tooling override: 0 | 1
    const int nch = (ncols + 63) / 64;
    bool want = passes * (nch - 1) >= 15;
    if (c->f64_engine == CORU_F64_OZAKI_PLANES) want = true;
    if (c->f64_engine == CORU_F64_OZAKI_INLINE || c->f64_engine == CORU_F64_OZAKI_HYBRID) want = false;
    if (planes_env) want = atoi(planes_env) != 0;
    if (want) {
        const OzPlaneDims pd = gemm_oz_plane_dims(rows, cols);
        const size_t need = pd.pn_bytes + pd.pt_bytes;
        bool fits = need <= c->oz_planes_cap;
        if (!fits) {
            size_t free_b = 0, total_b = 0;
            CORU_CUDA(cudaMemGetInfo(&free_b, &total_b));
            fits = need + (size_t(4) << 30) <= free_b + c->oz_planes_cap;
        }
        if (fits && ensure_dev(c, &c->oz_planes, &c->oz_planes_cap, need, "Ozaki digit planes") == CORU_OK) {
            CORU_CUDA(gemm_oz_planes(A, lda, rows, cols, c->oz_e, c->oz_e + rows, static_cast<uint8_t*>(c->oz_planes),
                                     c->stream));
            ++g_launches;
            c->oz_planes_ready = true;
        }
    }
    // Hybrid (no conversion pass): the first full op-N pass converts in the kernel and ALSO writes
    // the row-scaled planes (7 bytes per entry); the later op-N passes stream those. Op-T passes
    // keep the in-kernel conversion (the plane kernel is not faster there). Worth it from the
    // first re-use on (C3: a plane pass 1.47 instead of 1.69 ms, the storing pass +0.13 ms).
    static const char* hybrid_env = getenv("CORU_OZ_HYBRID");  // tooling override: 0 | 1
    bool hybrid = !c->oz_planes_ready && !want && passes_n >= 2;
    if (hybrid_env) hybrid = !c->oz_planes_ready && atoi(hybrid_env) != 0 && passes_n >= 2;
    if (c->f64_engine == CORU_F64_OZAKI_INLINE) hybrid = false;
    if (c->f64_engine == CORU_F64_OZAKI_HYBRID) hybrid = passes_n >= 2;
    if (hybrid) {
        const size_t need = gemm_oz_plane_dims(rows, cols).pn_bytes;
        bool fits = need <= c->oz_planes_cap;
        if (!fits) {
            size_t free_b = 0, total_b = 0;
            CORU_CUDA(cudaMemGetInfo(&free_b, &total_b));
            fits = need + (size_t(4) << 30) <= free_b + c->oz_planes_cap;
        }
        if (fits && ensure_dev(c, &c->oz_planes, &c->oz_planes_cap, need, "Ozaki digit planes") == CORU_OK)
            c->oz_pn_state = 1;
    }
    c->oz_a = A;
    c->oz_lda = lda;
    c->oz_rows = rows;
    c->oz_cols = cols;
    return CORU_OK;
}

// check_corutv_params (corutv.hpp:67-71) + the q check (corutv.hpp:81), same messages.
int check_params(int64_t m, int64_t n, int64_t ell, int q) {
    if (m < 1 || n < 1) return fail(CORU_EINVAL, "Matrix: dimensions must be positive");
    if (ell < 1) return fail(CORU_EINVAL, "corutv: ell must be >= 1");
    if (ell >= std::min(m, n)) return fail(CORU_EINVAL, "corutv: ell must be < min(rows, cols)");
    if (q < 0) return fail(CORU_EINVAL, "corutv: q must be >= 0");
    return CORU_OK;
}

// ---- per-dtype kernel dispatch ------------------------------------------------------------------
template <typename T>
int64_t gemm_ws(Op op, int64_t Mo, int64_t K, int N, int sms);
template <>
int64_t gemm_ws<double>(Op op, int64_t Mo, int64_t K, int N, int sms) {
    return plan_gemm_f64(op, Mo, K, N, sms).ws_elems;
}
template <>
int64_t gemm_ws<float>(Op op, int64_t Mo, int64_t K, int N, int sms) {
    const int64_t simt = plan_gemm_f32(op, Mo, K, N, sms).ws_elems;
    return gemm_tc32_eligible(Mo, K, N) ? std::max(simt, gemm_tc32_ws_elems(Mo, K, N, sms)) : simt;
}

// The tensor-core fp32 path takes A-pass-sized products (A streamed once per N-chunk); small
// products (the core, the lift) stay on the FFMA kernel.
bool use_tc32(const coru_ctx* c, Op op, const float* A, int64_t lda, int64_t Mo, int64_t K, int N) {
    if (c->f32_path == CORU_F32_SIMT) return false;
    if (!gemm_tc32_supported(op, A, lda, Mo, K, N)) return false;
    return c->f32_path == CORU_F32_TC || Mo * K >= (int64_t(1) << 22);
}

template <typename T>
int gemm(coru_ctx* c, Op op, const T* A, int64_t lda, const T* X, int64_t ldx, T* C, int64_t ldc, int64_t Mo,
         int64_t K, int N, T* ws, int64_t ws_elems);
int prof_begin(coru_ctx* c, cudaEvent_t* stop) {
    if (c->prof_used == c->prof_events.size()) {
        cudaEvent_t a, b;
        CORU_CUDA(cudaEventCreate(&a));
        CORU_CUDA(cudaEventCreate(&b));
        c->prof_events.emplace_back(a, b);
    }
    if (c->prof_shared.size() < c->prof_events.size()) c->prof_shared.resize(c->prof_events.size(), 0);
    c->prof_shared[c->prof_used] = c->prof_overlap ? 1 : 0;
    auto& ev = c->prof_events[c->prof_used++];
    CORU_CUDA(cudaEventRecord(ev.first, c->stream));
    *stop = ev.second;
    return CORU_OK;
}

template <>
int gemm<double>(coru_ctx* c, Op op, const double* A, int64_t lda, const double* X, int64_t ldx, double* C,
                 int64_t ldc, int64_t Mo, int64_t K, int N, double* ws, int64_t ws_elems) {
    // A-passes over the prepared matrix: INT8 tensor cores (Ozaki), when the shape qualifies.
    if (c->oz_a && A == c->oz_a && lda == c->oz_lda &&
        (op == Op::N ? (Mo <= c->oz_rows && K == c->oz_cols) : (Mo == c->oz_cols && K <= c->oz_rows)) &&
        gemm_oz_supported(op, A, lda, Mo, K, N)) {
        CORU_TRY(ensure_dev(c, &c->oz_ws, &c->oz_ws_bytes, gemm_oz_ws_bytes(Mo, K, N, c->num_sms), "Ozaki workspace"));
        cudaEvent_t stop = nullptr;
        if (c->prof) CORU_TRY(prof_begin(c, &stop));
        const int* eA = op == Op::N ? c->oz_e : c->oz_e + c->oz_rows;
        OzPlanes pl;
        const bool use_pl = c->oz_planes_ready || (op == Op::N && c->oz_pn_state == 2);
        const bool store_pl = !use_pl && op == Op::N && c->oz_pn_state == 1 && Mo == c->oz_rows;
        if (use_pl || store_pl) {
            const OzPlaneDims pd = gemm_oz_plane_dims(c->oz_rows, c->oz_cols);
            const uint8_t* base = static_cast<const uint8_t*>(c->oz_planes);
            pl.p = op == Op::N ? base : base + pd.pn_bytes;
            pl.ld = op == Op::N ? pd.ldn : pd.ldt;
            pl.rows = op == Op::N ? c->oz_rows : c->oz_cols;
        }
        CORU_CUDA(gemm_oz(op, A, lda, use_pl ? &pl : nullptr, eA, X, ldx, C, ldc, Mo, K, N, c->oz_ws, c->num_sms,
                          c->stream, store_pl ? &pl : nullptr));
        if (store_pl) c->oz_pn_state = 2;
        c->last_f64_engine = c->oz_planes_ready ? 2 : (c->oz_pn_state ? 3 : 1);
        if (stop) {
            CORU_CUDA(cudaEventRecord(stop, c->stream));
            c->prof_flops += 2.0 * double(Mo) * double(K) * double(N);
            c->prof_bytes += 8.0 * double(Mo) * double(K);
        }
        g_launches += gemm_oz_launches(Mo, K, N, c->num_sms);
        return CORU_OK;
    }
    GemmPlan p = plan_gemm_f64(op, Mo, K, N, c->num_sms);
    if (p.ws_elems > ws_elems) return fail(CORU_ECUDA, "internal: gemm workspace too small");
    cudaEvent_t stop = nullptr;
    if (c->prof) CORU_TRY(prof_begin(c, &stop));
    CORU_CUDA(gemm_f64(op, A, lda, X, ldx, C, ldc, Mo, K, N, p, ws, c->stream));
    if (stop) {
        CORU_CUDA(cudaEventRecord(stop, c->stream));
        c->prof_flops += 2.0 * double(Mo) * double(K) * double(N);
        c->prof_bytes += 8.0 * double(Mo) * double(K);
    }
    g_launches += 1;  // stream-K fix-up runs inside the GEMM
    return CORU_OK;
}
template <>
int gemm<float>(coru_ctx* c, Op op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C, int64_t ldc,
                int64_t Mo, int64_t K, int N, float* ws, int64_t ws_elems) {
    const bool tc = use_tc32(c, op, A, lda, Mo, K, N);
    GemmPlan p = plan_gemm_f32(op, Mo, K, N, c->num_sms);
    const int64_t need = tc ? gemm_tc32_ws_elems(Mo, K, N, c->num_sms) : p.ws_elems;
    if (need > ws_elems) return fail(CORU_ECUDA, "internal: gemm workspace too small");
    cudaEvent_t stop = nullptr;
    if (c->prof) CORU_TRY(prof_begin(c, &stop));
    if (tc)
        CORU_CUDA(gemm_tc32(op, A, lda, X, ldx, C, ldc, Mo, K, N, ws, c->num_sms, c->max_smem, c->stream));
    else
        CORU_CUDA(gemm_f32(op, A, lda, X, ldx, C, ldc, Mo, K, N, p, ws, c->stream));
    if (stop) {
        CORU_CUDA(cudaEventRecord(stop, c->stream));
        c->prof_flops += 2.0 * double(Mo) * double(K) * double(N);
        c->prof_bytes += 4.0 * double(Mo) * double(K);
    }
    g_launches += tc ? gemm_tc32_launches(Mo, K, N, c->num_sms) : (p.splits > 1 ? 2 : 1);
    return CORU_OK;
}

template <typename T>
struct TsqrBufs {
    TsqrPlan plan;
    T *v = nullptr, *beta = nullptr, *tarena = nullptr, *rarena = nullptr, *scratch = nullptr;
    int max_smem = 0, sms = 148;
    // Wide sketches: CholeskyQR2 in fp64 first; the Householder tree is gated on its status.
    bool chol = false;
    CholQrPlan cp;
    double* cws = nullptr;
    int* status = nullptr;
    void carve(Carver& cv, int64_t rows, int d, int smem, int num_sms = 148, bool allow_chol = false) {
        max_smem = smem;
        sms = num_sms;
        plan = plan_tsqr(rows, d, sizeof(T), smem, num_sms);
        v = cv.take<T>(plan.v_elems);
        beta = cv.take<T>(plan.beta_elems);
        tarena = cv.take<T>(plan.t_elems);
        rarena = cv.take<T>(plan.r_elems);
        scratch = cv.take<T>(tsqr_scratch_elems(plan));
        chol = allow_chol && cholqr_applicable(rows, d, smem);
        if (chol) {
            cp = plan_cholqr(rows, d, sizeof(T), num_sms);
            cws = cv.take<double>(cholqr_ws_doubles(cp));
            status = cv.take<int>(1);
        }
    }
    // ext_gate: another tree's CholeskyQR2 status gating THIS tree (the cross-rank top level of a
    // sharded wide sketch runs only when the sharded CholeskyQR2 fell back).
    const int* ext_gate = nullptr;
    const int* gate() const { return chol ? status : ext_gate; }
    // CholeskyQR2 alone (reduce: the cross-rank sum of the Gram matrices of a row-sharded sketch).
    int factor_chol(const T* B, int64_t ldb, T* r_out, cudaStream_t st, const CholQrReduce* reduce = nullptr) {
        CORU_CUDA(cholqr_factor<T>(cp, B, ldb, cws, status, r_out, max_smem, sms, st, reduce));
        g_launches += cholqr_launches(plan.d);
        return CORU_OK;
    }
    // The Householder tree alone (gated on the CholeskyQR2 status when there is one).
    int factor_tree(const T* B, int64_t ldb, T* r_out, cudaStream_t st) {
        CORU_CUDA(tsqr_factor<T>(plan, B, ldb, v, beta, tarena, rarena, r_out, st, gate()));
        g_launches += int64_t(plan.levels.size());
        return CORU_OK;
    }
    int factor(const T* B, int64_t ldb, T* r_out, cudaStream_t st) {
        if (chol) CORU_TRY(factor_chol(B, ldb, r_out, st));
        return factor_tree(B, ldb, r_out, st);
    }
    int form_q_chol(T* Q, int64_t ldq, cudaStream_t st) {
        CORU_CUDA(cholqr_form_q<T>(cp, cws, Q, ldq, sms, st));
        ++g_launches;
        return CORU_OK;
    }
    int form_q_tree(const T* q_top, T* Q, int64_t ldq, cudaStream_t st) {
        CORU_CUDA(tsqr_form_q<T>(plan, q_top, v, beta, tarena, scratch, Q, ldq, max_smem, st, gate()));
        g_launches += int64_t(plan.levels.size());
        return CORU_OK;
    }
    int form_q(const T* q_top, T* Q, int64_t ldq, cudaStream_t st) {
        if (chol) {
            if (q_top) return fail(CORU_ECUDA, "internal: CholeskyQR2 tree with a top-level Q");
            CORU_TRY(form_q_chol(Q, ldq, st));
        }
        return form_q_tree(q_top, Q, ldq, st);
    }
};

enum class Mode { Full, Sketch, Project };

// One decomposition request, already mapped onto A' (= A, or A^T for the ULV orientation).
template <typename T>
struct Request {
    const T* A = nullptr;
    int64_t lda = 0;
    bool trans = false;     // run on A' = A^T (corutv.hpp:82-87), zero-copy via the op flag
    int64_t rows = 0;       // rows of A' held by this rank
    int64_t cols = 0;       // cols of A'
    int d = 0;
    int q = 0;
    uint64_t seed = 0, stream = 0;
    Mode mode = Mode::Full;
    bool first_done = false;  // the first power round (Φ, c1 = a·Φ, c2 = a^T·c1) is already in the workspace
    // Stream capture (run_graph): Φ already sits in the pinned staging buffer, the flag / pivots go to
    // the context's pinned host slots, and nothing synchronises — the caller launches the graph.
    bool capture = false;
    int variant = CORU_D_EXACT;  // Full: how D is formed (corutv.hpp:89-92)
    // Full: U' (rows x d), T' (d x d), V' (cols x d) — device, caller's buffers.
    T* u = nullptr;
    int64_t ldu = 0;
    T* t = nullptr;
    int64_t ldt = 0;
    bool t_transpose = false;
    T* v = nullptr;
    int64_t ldv = 0;
    int64_t* perm_host = nullptr;
    int* warn_host = nullptr;
    // Out-of-core (§8 f4): A' stays in host memory (row-major, lda) and is streamed in row chunks
    // of ooc_rows rows; A must then be null. Single GPU, rows >= cols.
    const T* a_host = nullptr;
    int64_t ooc_rows = 0;
    // Sketch: Q1, Q2, C1, C2prev (device, may be null except Q1/Q2).
    T *q1 = nullptr, *q2 = nullptr, *c1 = nullptr, *c2p = nullptr;
    int64_t ldq1 = 0, ldq2 = 0, ldc1 = 0, ldc2 = 0;
    Op op_a() const { return trans ? Op::T : Op::N; }   // A'·X
    Op op_at() const { return trans ? Op::N : Op::T; }  // A'^T·Y
};

// Sharded power rounds: B2 = sum_g A_g^T B1_g is an all-reduce of n x d per round (C4 58 MB, C5 136 MB).
// Worth hiding when it is large: the product is then issued per 64-column chunk of the sketch and
// each chunk's sum runs on the aux stream while the next chunk's GEMM runs.
constexpr int kB2ChunkCols = 64;
inline bool overlap_b2(const coru_ctx* c, int64_t n, int dp, size_t elem) {
    const char* env = getenv("CORU_B2_OVERLAP");  // tooling / tests: 0 | 1 (read per call)
    if (env) return atoi(env) != 0 && c->world > 1 && dp > kB2ChunkCols;
    return c->world > 1 && dp > kB2ChunkCols && size_t(n) * size_t(dp) * elem >= (size_t(8) << 20);
}

template <typename T>
struct Work {
    T *b2 = nullptr, *b2prev = nullptr, *b1 = nullptr, *q1 = nullptr, *q2 = nullptr, *gws = nullptr;
    int64_t gws_elems = 0;
    TsqrBufs<T> ts1, ts2, tstop;
    T *rstack = nullptr, *qtop = nullptr, *r1loc = nullptr, *r1 = nullptr, *r2 = nullptr;
    T *m = nullptr, *qm = nullptr, *tm = nullptr, *qrcp_scr = nullptr;
    T *y1 = nullptr, *y2 = nullptr, *pinv = nullptr;  // approx-D core
    T *cbuf[2] = {nullptr, nullptr}, *b2n = nullptr, *part = nullptr;  // out-of-core chunk ring, next c2, partial
    T* tnp = nullptr;  // partials of the skinny Q^T·W core products (d <= 64)
    T* wproj = nullptr;  // W = A·Q2 when it overlaps the Q1 tree (exact-D, single GPU, in-core)
    T* b2chunks = nullptr;  // sharded: contiguous column chunks of A_g^T·B1_g, all-reduced chunk by chunk
    double* pws = nullptr;
    int64_t* perm = nullptr;
    int* flag = nullptr;

    void layout(Carver& cv, const coru_ctx* c, const Request<T>& r, int dp) {
        const int64_t R = r.rows, N = r.cols;
        const int d = r.d, sms = c->num_sms;
        b2 = cv.take<T>(N * dp);
        const bool approx = r.mode == Mode::Full && r.variant == CORU_D_APPROX;
        b2prev = (r.c2p || approx) ? cv.take<T>(N * dp) : nullptr;
        b1 = cv.take<T>(R * dp);
        q1 = cv.take<T>(R * dp);
        q2 = cv.take<T>(N * dp);
        gws_elems = std::max({gemm_ws<T>(r.op_a(), R, N, d, sms), gemm_ws<T>(r.op_at(), N, R, d, sms),
                              gemm_ws<T>(Op::T, d, R, d, sms), gemm_ws<T>(Op::N, R, d, d, sms),
                              gemm_ws<T>(Op::T, d, N, d, sms), gemm_ws<T>(Op::N, d, d, d, sms)});
        if (overlap_b2(c, N, dp, sizeof(T)))  // the per-chunk A^T-products of the sharded power rounds
            for (int nc : {std::min(kB2ChunkCols, d), d % kB2ChunkCols ? d % kB2ChunkCols : std::min(kB2ChunkCols, d)})
                gws_elems = std::max(gws_elems, gemm_ws<T>(r.op_at(), N, R, nc, sms));
        if (std::is_same<T, float>::value && N * int64_t(d) >= (int64_t(1) << 22))  // the sketch over Φ row chunks (run_impl)
            for (int64_t kk : {N / 8 - 4, N / 8, N / 8 + 4, N - 7 * (N / 8) + 28})
                gws_elems = std::max(gws_elems, gemm_ws<T>(Op::N, R, kk, d, sms));
        if (r.a_host) {
            // host rows of A: rows of A' (URV) or its columns (ULV, A' = A^T); row length = the other side
            const int64_t HR = r.trans ? N : R, HL = r.trans ? R : N;
            const int64_t cr = std::min(r.ooc_rows, HR), last = HR - (HR - 1) / cr * cr;
            for (int64_t rows : {cr, last})
                gws_elems = std::max({gws_elems, gemm_ws<T>(Op::N, rows, HL, d, sms), gemm_ws<T>(Op::T, HL, rows, d, sms)});
            cbuf[0] = cv.take<T>(cr * HL);
            cbuf[1] = cv.take<T>(cr * HL);
            b2n = cv.take<T>(N * dp);
            part = cv.take<T>(HL * dp);
        }
        gws = cv.take<T>(gws_elems);
        // CholeskyQR2 for wide sketches; sharded, the Gram matrices of Q1's sketch are summed over the
        // ranks and the cross-rank Householder top level is gated on its status
        ts1.carve(cv, R, d, c->max_smem, sms, c->wide_qr);
        ts2.carve(cv, N, d, c->max_smem, sms, c->wide_qr);
        if (c->world > 1) {
            // column chunks of the A^T-product, reduced on the aux stream under the next chunk's GEMM
            if (overlap_b2(c, N, dp, sizeof(T))) b2chunks = cv.take<T>(N * int64_t(dp));
            rstack = cv.take<T>(int64_t(c->world) * d * d);
            tstop.carve(cv, int64_t(c->world) * d, d, c->max_smem);
            tstop.ext_gate = ts1.chol ? ts1.status : nullptr;
            qtop = cv.take<T>(int64_t(c->world) * d * d);
        }
        r1loc = cv.take<T>(int64_t(d) * d);
        r1 = cv.take<T>(int64_t(d) * d);
        r2 = cv.take<T>(int64_t(d) * d);
        m = cv.take<T>(int64_t(d) * dp);
        if (d <= 64) tnp = cv.take<T>(int64_t(kTnMaxBlocks) * d * d);
        if (r.mode == Mode::Full && r.variant != CORU_D_APPROX && c->world == 1 && !r.a_host &&
            getenv("CORU_EARLY_JOIN") == nullptr)
            wproj = cv.take<T>(R * dp);
        qm = cv.take<T>(int64_t(dp) * dp);
        tm = cv.take<T>(int64_t(d) * d);
        qrcp_scr = cv.take<T>(qrcp_scratch_elems(d));
        if (approx) {
            y1 = cv.take<T>(int64_t(d) * dp);
            y2 = cv.take<T>(int64_t(d) * dp);
            pinv = cv.take<T>(int64_t(d) * dp);
            pws = cv.take<double>(pinv_ws_doubles(d));
        }
        perm = cv.take<int64_t>(d);
        flag = cv.take<int>(4);
    }
};

template <typename T>
__global__ void k_sum_slots(const T* const* slots, int world, T* out, size_t count) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += size_t(gridDim.x) * blockDim.x) {
        T s = slots[0][e];
        for (int r = 1; r < world; ++r) s += slots[r][e];  // rank order: identical bytes on every rank
        out[e] = s;
    }
}

template <typename T>
int thread_allreduce(coru_ctx* c, T* buf, size_t count, cudaStream_t stream) {
    coru_threadcomm* g = c->tcomm;
    const size_t bytes = count * sizeof(T) + size_t(g->world) * sizeof(void*);
    if (c->tscratch_bytes < bytes) {
        CORU_CUDA(cudaStreamSynchronize(stream));
        if (c->tscratch) cudaFree(c->tscratch);
        c->tscratch = nullptr;
        c->tscratch_bytes = 0;
        if (cudaMalloc(&c->tscratch, bytes) != cudaSuccess) return fail(CORU_ENOMEM, "thread-comm scratch");
        c->tscratch_bytes = bytes;
    }
    CORU_CUDA(cudaStreamSynchronize(stream));
    g->slots[size_t(c->rank)] = buf;
    if (!g->barrier()) return fail(CORU_ECUDA, "a peer rank of the thread group failed");
    const T** dslots = reinterpret_cast<const T**>(static_cast<char*>(c->tscratch) + count * sizeof(T));
    CORU_CUDA(cudaMemcpyAsync(dslots, g->slots.data(), size_t(g->world) * sizeof(void*), cudaMemcpyHostToDevice,
                              stream));
    T* tmp = static_cast<T*>(c->tscratch);
    const int blocks = int(std::min<size_t>((count + 255) / 256, 148 * 8));
    k_sum_slots<T><<<std::max(blocks, 1), 256, 0, stream>>>(dslots, g->world, tmp, count);
    ++g_launches;
    CORU_CUDA(cudaGetLastError());
    CORU_CUDA(cudaStreamSynchronize(stream));
    if (!g->barrier()) return fail(CORU_ECUDA, "a peer rank of the thread group failed");
    CORU_CUDA(cudaMemcpyAsync(buf, tmp, count * sizeof(T), cudaMemcpyDeviceToDevice, stream));
    return CORU_OK;
}

template <typename T>
int thread_allgather(coru_ctx* c, const T* send, T* recv, size_t count) {
    coru_threadcomm* g = c->tcomm;
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    g->slots[size_t(c->rank)] = send;
    if (!g->barrier()) return fail(CORU_ECUDA, "a peer rank of the thread group failed");
    for (int r = 0; r < g->world; ++r)
        CORU_CUDA(cudaMemcpyAsync(recv + size_t(r) * count, g->slots[size_t(r)], count * sizeof(T),
                                  cudaMemcpyDeviceToDevice, c->stream));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    if (!g->barrier()) return fail(CORU_ECUDA, "a peer rank of the thread group failed");
    return CORU_OK;
}

template <typename T>
int allreduce(coru_ctx* c, T* buf, size_t count, cudaStream_t stream = nullptr) {
    if (c->world <= 1 && !c->comm) return CORU_OK;
    if (!stream) stream = c->stream;
    if (c->tcomm) return thread_allreduce<T>(c, buf, count, stream);
    CORU_NCCL(nccl()->AllReduce(buf, buf, count, nccl_type<T>(), ncclSum, c->comm, stream));
    return CORU_OK;
}

template <typename T>
int allgather(coru_ctx* c, const T* send, T* recv, size_t count) {
    if (c->tcomm) return thread_allgather<T>(c, send, recv, count);
    CORU_NCCL(nccl()->AllGather(send, recv, count, nccl_type<T>(), c->comm, c->stream));
    return CORU_OK;
}

// Φ = gaussian(rows, cols, {seed, stream}) generated on the host with the host libm (bit-identical
// to the reference's gaussian(), rng.hpp:86-112) into the pinned staging buffer, in row chunks:
// chunk i+1 is generated by the worker pool while the DMA engine uploads chunk i on `st`.
// Chunk boundaries start on Box–Muller pairs (row·cols even).
// Start generating gaussian(rows, cols, {seed, stream}) (padded to ld) in the background; the next
// upload_phi_host with exactly these parameters takes it, any other discards it.
template <typename T>
int phi_prefetch(coru_ctx* c, int64_t rows, int cols, int ld, uint64_t seed, uint64_t stream) {
    if (c->phi_mode != CORU_PHI_HOST_EXACT) return CORU_OK;
    if (c->pf_thread.joinable()) c->pf_thread.join();
    c->pf_active = false;
    const size_t bytes = size_t(rows) * ld * sizeof(T);
    if (bytes > c->pf_bytes) {
        CORU_CUDA(cudaEventSynchronize(c->ev_pf));
        if (c->pf_buf) cudaFreeHost(c->pf_buf);
        c->pf_buf = nullptr;
        c->pf_bytes = 0;
        if (cudaMallocHost(&c->pf_buf, bytes) != cudaSuccess) {
            cudaGetLastError();
            return CORU_OK;  // no prefetch: the regular path generates it
        }
        c->pf_bytes = bytes;
    }
    CORU_CUDA(cudaEventSynchronize(c->ev_pf));  // the last copy out of the buffer has drained
    c->pf_seed = seed;
    c->pf_stream = stream;
    c->pf_rows = rows;
    c->pf_cols = cols;
    c->pf_ld = ld;
    c->pf_elem = sizeof(T);
    T* buf = reinterpret_cast<T*>(c->pf_buf);
    const int threads = c->host_threads;
    c->pf_thread = std::thread([=] { gaussian_host_rows<T>(rows, cols, seed, stream, buf, ld, threads, 1, 0, rows); });
    c->pf_active = true;
    return CORU_OK;
}

// on_chunk(r0, r1), if given, is called after the upload of rows [r0, r1) has been enqueued on st
// (r0 a multiple of 4): the caller's work on those rows then runs while the host generates the next.
using PhiChunkFn = std::function<int(int64_t, int64_t)>;
template <typename T>
int upload_phi_host(coru_ctx* c, int64_t rows, int cols, int ld, uint64_t seed, uint64_t stream, T* out,
                    cudaStream_t st, const PhiChunkFn* on_chunk = nullptr) {
    const size_t bytes = size_t(rows) * ld * sizeof(T);
    if (c->pf_active) {
        c->pf_thread.join();
        c->pf_active = false;
        if (c->pf_seed == seed && c->pf_stream == stream && c->pf_rows == rows && c->pf_cols == cols && c->pf_ld == ld &&
            c->pf_elem == sizeof(T)) {
            CORU_CUDA(cudaMemcpyAsync(out, c->pf_buf, bytes, cudaMemcpyHostToDevice, st));
            CORU_CUDA(cudaEventRecord(c->ev_pf, st));
            return on_chunk ? (*on_chunk)(0, rows) : CORU_OK;
        }
    }
    CORU_TRY(ensure_pinned(c, bytes));
    // The pinned staging buffer is reused across calls: wait for the LAST copy out of it only (not
    // for the stream — the exponent / digit-plane kernels of this call keep running while the host
    // generates Φ).
    CORU_CUDA(cudaEventSynchronize(c->ev_phi));
    T* phi = reinterpret_cast<T*>(c->pinned);
    const int64_t total = rows * int64_t(cols);
    const int chunks = int(std::max<int64_t>(1, std::min<int64_t>(8, total / (1 << 17))));
    int64_t r0 = 0;
    for (int k = 1; k <= chunks; ++k) {
        int64_t r1 = k == chunks ? rows : rows * k / chunks;
        if (k < chunks && ((r1 * cols) & 1)) --r1;  // odd cols: end on an even row so the next chunk starts on a pair
        if (k < chunks && on_chunk) r1 &= ~int64_t(3);  // 16-byte aligned sub-matrices for the caller (still even)
        if (r1 <= r0) continue;
        gaussian_host_rows<T>(rows, cols, seed, stream, phi, ld, c->host_threads, 1, r0, r1);
        CORU_CUDA(cudaMemcpyAsync(out + r0 * ld, phi + r0 * ld, size_t(r1 - r0) * ld * sizeof(T),
                                  cudaMemcpyHostToDevice, st));
        if (on_chunk) CORU_TRY((*on_chunk)(r0, r1));
        r0 = r1;
    }
    CORU_CUDA(cudaEventRecord(c->ev_phi, st));
    return CORU_OK;
}

// Φ = gaussian(cols, ell, seed), padded to dp columns (corutv.hpp:51). Default: host-generated,
// bit-exact (upload_phi_host). CORU_PHI_DEVICE (opt-in): the device generator (same word stream,
// device log/sincos, a few ulp off).
template <typename T>
int gen_phi(coru_ctx* c, const Request<T>& r, T* out, int dp, const PhiChunkFn* on_chunk = nullptr) {
    const int64_t N = r.cols;
    cudaStream_t st = c->stream;
    if (c->phi_mode == CORU_PHI_DEVICE) {
        uint64_t s4[4];
        seed_state_words(r.seed, r.stream, s4);
        CORU_CUDA(gaussian_dev<T>(N, r.d, s4, out, dp, st));
        ++g_launches;
        return on_chunk ? (*on_chunk)(0, N) : CORU_OK;
    }
    return upload_phi_host<T>(c, N, r.d, dp, r.seed, r.stream, out, st, on_chunk);
}

template <typename T>
int run_impl(coru_ctx* c, const Request<T>& r, size_t extra_arena_off);

// The hot path. Enqueues everything on c->stream and synchronises once at the end (the flag and
// Skinny transposed product C (d x d) = Q^T·W for Q, W m x d (ld dp), d <= 64: the core
// Q1^T·(A·Q2) and the approx-D cores Q1^T·c1, Q2^T·c2prev. The stream-K GEMM splits each of its one
// or two output tiles over ~60 CTAs whose partials one owner sums serially (53 us at C2); here each
// CTA reduces a row block into a private d x d partial (4x4 register tile per thread, rows staged
// through shared memory) and one fixed-order pass sums the partials: deterministic, ~8 us.
constexpr int kTnRows = 32;
template <typename T>
__global__ void __launch_bounds__(256) k_tn_partial(const T* __restrict__ Q, int64_t ldq, const T* __restrict__ W,
                                                    int64_t ldw, int64_t m, int d, int64_t rows_per_blk,
                                                    T* __restrict__ part) {
    __shared__ __align__(16) T sQ[kTnRows][64];
    __shared__ __align__(16) T sW[kTnRows][64];
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;  // rows 4ti.., cols 4tj.. of the output
    const int64_t r0 = int64_t(blockIdx.x) * rows_per_blk, r1 = min(m, r0 + rows_per_blk);
    T acc[4][4] = {};
    for (int64_t rb = r0; rb < r1; rb += kTnRows) {
        for (int e = threadIdx.x; e < kTnRows * 64; e += 256) {
            const int r = e >> 6, c = e & 63;
            const bool ok = rb + r < r1 && c < d;
            sQ[r][c] = ok ? Q[(rb + r) * ldq + c] : T(0);
            sW[r][c] = ok ? W[(rb + r) * ldw + c] : T(0);
        }
        __syncthreads();
#pragma unroll 4
        for (int r = 0; r < kTnRows; ++r) {
            T a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = sQ[r][4 * ti + u];
                b[u] = sW[r][4 * tj + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
    T* out = part + int64_t(blockIdx.x) * d * d;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int i = 4 * ti + u, j = 4 * tj + v;
            if (i < d && j < d) out[i * d + j] = acc[u][v];
        }
}
// 32 outputs per CTA (one per lane); the 8 warps sum contiguous eighths of the partials, then the
// eight warp sums are added in warp order: a fixed order, so the result is deterministic.
template <typename T>
__global__ void __launch_bounds__(256) k_tn_reduce(const T* __restrict__ part, int nblk, int d, T* __restrict__ C,
                                                   int64_t ldc) {
    __shared__ T ws[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int e = blockIdx.x * 32 + lane;
    const int per = (nblk + 7) / 8, b0 = warp * per, b1 = min(nblk, b0 + per);
    T s = T(0);
    if (e < d * d) {
#pragma unroll 4
        for (int b = b0; b < b1; ++b) s += part[int64_t(b) * d * d + e];
    }
    ws[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && e < d * d) {
        T t = ws[0][lane];
        for (int w = 1; w < 8; ++w) t += ws[w][lane];
        C[int64_t(e / d) * ldc + e % d] = t;
    }
}
template <typename T>
int tn_small(coru_ctx* c, const T* Q, int64_t ldq, const T* W, int64_t ldw, int64_t m, int d, T* C, int64_t ldc,
             T* part) {
    const int64_t want = (m + kTnRows - 1) / kTnRows;  // one staged chunk per CTA (C2: 125 CTAs)
    const int nblk = int(std::max<int64_t>(1, std::min<int64_t>(want, kTnMaxBlocks)));
    const int64_t rpb = (m + nblk - 1) / nblk;
    k_tn_partial<T><<<nblk, 256, 0, c->stream>>>(Q, ldq, W, ldw, m, d, rpb, part);
    k_tn_reduce<T><<<(d * d + 31) / 32, 256, 0, c->stream>>>(part, nblk, d, C, ldc);
    g_launches += 2;
    CORU_CUDA(cudaGetLastError());
    return CORU_OK;
}
// Q^T·W (d x d): the skinny kernel for d <= 64 (CORU_TN_SMALL=0 restores the GEMM), else the GEMM.
template <typename T>
int gemm_tn_core(coru_ctx* c, const T* Q, int64_t ldq, const T* W, int64_t ldw, int64_t m, int d, T* C, int64_t ldc,
                 T* part, T* gws, int64_t gws_elems) {
    static const bool on = getenv("CORU_TN_SMALL") == nullptr || atoi(getenv("CORU_TN_SMALL")) != 0;
    if (on && part && d <= 64) return tn_small<T>(c, Q, ldq, W, ldw, m, d, C, ldc, part);
    return gemm<T>(c, Op::T, Q, ldq, W, ldw, C, ldc, d, m, d, gws, gws_elems);
}

template <typename T>
__global__ void k_add_inplace(T* __restrict__ dst, const T* __restrict__ src, size_t count) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += size_t(gridDim.x) * blockDim.x)
        dst[e] += src[e];
}
template <typename T>
cudaError_t add_inplace(T* dst, const T* src, size_t count, cudaStream_t st) {
    const int blocks = int(std::min<size_t>((count + 255) / 256, 148 * 8));
    k_add_inplace<T><<<std::max(blocks, 1), 256, 0, st>>>(dst, src, count);
    return cudaGetLastError();
}

// the pivots are host outputs). A failing rank of an in-process group releases its peers.
template <typename T>
int run(coru_ctx* c, const Request<T>& r, size_t extra_arena_off = 0) {
    if constexpr (std::is_same<T, double>::value) {
        if (r.A) {  // device-resident A: the stored matrix is rows x cols, or its transpose (ULV)
            const int passes = r.mode == Mode::Sketch ? 2 * r.q + 2 : 2 * r.q + (r.variant == CORU_D_APPROX ? 2 : 3);
            // op-N passes over the STORED matrix: a·c2 products (q + 1, + a·q2 for exact D) when it is
            // A itself, the q + 1 a^T·c1 products when it holds the transpose; minus the one the host
            // entry already ran chunk by chunk
            int passes_n = r.trans ? r.q + 1 : passes - (r.q + 1);
            if (r.first_done) --passes_n;
            const int rc = oz_prepare(c, r.A, r.lda, r.trans ? r.cols : r.rows, r.trans ? r.rows : r.cols, passes, r.d,
                                      passes_n);
            if (rc != CORU_OK) {
                if (c->tcomm) c->tcomm->abort();
                return rc;
            }
        }
    }
    const int rc = run_impl<T>(c, r, extra_arena_off);
    c->oz_a = nullptr;
    if (rc != CORU_OK && c->tcomm) c->tcomm->abort();
    return rc;
}

template <typename T>
int run_impl(coru_ctx* c, const Request<T>& r, size_t extra_arena_off) {
    const int d = r.d;
    const int dp = int(round_up(d, 8));
    const int64_t R = r.rows, N = r.cols;
    cudaStream_t st = c->stream;
    Work<T> w;
    Carver meas{nullptr, extra_arena_off};
    w.layout(meas, c, r, dp);
    CORU_TRY(ensure_arena(c, meas.off));
    Carver cv{c->arena, extra_arena_off};
    w.layout(cv, c, r, dp);

    // Φ = gaussian(cols, ell, seed), padded to dp columns (corutv.hpp:51): on the device, or on the
    // host with the host libm (bit-exact) and one H2D.
    CORU_CUDA(cudaMemsetAsync(w.q1, 0, size_t(R) * dp * sizeof(T), st));
    CORU_CUDA(cudaMemsetAsync(w.q2, 0, size_t(N) * dp * sizeof(T), st));
    // A large Φ costs the host tens of milliseconds (C5: 34 M Gaussians, ~25 ms on 16 threads) during
    // which a pass that needs all of it would leave the GPU idle. fp32 (no exponent / digit pre-pass
    // to hide it under): the sketch c1 = a·Φ is accumulated over the row chunks of Φ as they arrive —
    // a[:, r0:r1]·Φ[r0:r1, :] per chunk, summed in chunk order (q1 is the scratch; its d columns are
    // rewritten by the explicit Q1 later) — so the GPU trails the generator by one chunk.
    // CORU_PHI_SEGMENTS=0/1 overrides (tooling).
    bool sketch_done = false;
    if (r.capture) {
        CORU_CUDA(cudaMemcpyAsync(w.b2, c->pinned, size_t(N) * dp * sizeof(T), cudaMemcpyHostToDevice, st));
    } else if (!r.first_done) {
        static const char* seg_env = getenv("CORU_PHI_SEGMENTS");
        bool seg = std::is_same<T, float>::value && r.A && !r.trans && !r.a_host && c->phi_mode == CORU_PHI_HOST_EXACT &&
                   N * int64_t(d) >= (int64_t(1) << 22);
        if (seg_env) seg = seg && atoi(seg_env) != 0;
        if (seg) {
            const PhiChunkFn on_chunk = [&](int64_t r0, int64_t r1) -> int {
                T* out = r0 == 0 ? w.b1 : w.q1;
                CORU_TRY(gemm<T>(c, Op::N, r.A + r0, r.lda, w.b2 + r0 * dp, dp, out, dp, R, r1 - r0, d, w.gws, w.gws_elems));
                if (r0 > 0) {
                    CORU_CUDA(add_inplace<T>(w.b1, w.q1, size_t(R) * dp, st));
                    ++g_launches;
                }
                return CORU_OK;
            };
            CORU_TRY(gen_phi<T>(c, r, w.b2, dp, &on_chunk));
            sketch_done = true;
        } else {
            CORU_TRY(gen_phi<T>(c, r, w.b2, dp));
        }
    }

    // Sketch and power rounds (corutv.hpp:54-58): c1 = a·c2 ; c2_prev = c2 ; c2 = a^T·c1.
    // The two QRs are independent and latency-bound (one CTA per tree block), so they run on two
    // streams: single-GPU, QR(c1) starts on the aux stream as soon as the last c1 exists and
    // overlaps the last A^T pass; with a communicator QR(c1) stays on the main stream (its
    // all-gather must keep the NCCL issue order) and QR(c2) goes to the aux stream.
    const bool sharded = c->world > 1;
    // Tall sketches (rows >= 16 cols: C3): QR(c1) is the critical path after the passes, so its tree
    // starts as soon as the last c1 exists and overlaps the last A^T pass — the upper tree levels
    // occupy a few SMs only (C3: 14.2 -> 13.6 ms). Square-ish problems keep both trees after the
    // pass (overlapping only slowed it there). CORU_QR1_EARLY=0/1 overrides (tooling).
    static const char* early_env = getenv("CORU_QR1_EARLY");
    const bool early_want = early_env ? atoi(early_env) != 0 : R >= 16 * N;
    const bool early_qr1 = !sharded && !r.a_host && early_want && !(r.first_done && r.q == 0);
    // Out-of-core: stream A' through a two-buffer device ring, H2D on the aux stream one chunk ahead
    // of the GEMMs on the main stream (events order the reuse of each buffer).
    cudaEvent_t ooc_ev[4] = {};
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            for (int i = 0; i < 4; ++i)
                if (e[i]) cudaEventDestroy(e[i]);
        }
    } ooc_guard{ooc_ev};
    if (r.a_host) {
        for (auto& e : ooc_ev) CORU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CORU_CUDA(cudaMemsetAsync(w.b2n, 0, size_t(N) * dp * sizeof(T), st));  // padding columns stay zero
        CORU_CUDA(cudaMemsetAsync(w.part, 0, size_t(r.trans ? R : N) * dp * sizeof(T), st));
    }
    const int64_t HR = r.trans ? N : R, HL = r.trans ? R : N;  // host rows of A, their length
    auto stream_a = [&](auto&& on_chunk) -> int {
        const int64_t cr = std::min(r.ooc_rows, HR);
        const int64_t nch = (HR + cr - 1) / cr;
        auto issue = [&](int64_t i) -> int {
            const int64_t r0 = i * cr, rows = std::min(cr, HR - r0);
            const int b = int(i & 1);
            CORU_CUDA(cudaStreamWaitEvent(c->aux, ooc_ev[2 + b], 0));  // buffer b free again
            CORU_CUDA(cudaMemcpy2DAsync(w.cbuf[b], size_t(HL) * sizeof(T), r.a_host + r0 * r.lda,
                                        size_t(r.lda) * sizeof(T), size_t(HL) * sizeof(T), size_t(rows),
                                        cudaMemcpyHostToDevice, c->aux));
            CORU_CUDA(cudaEventRecord(ooc_ev[b], c->aux));
            return CORU_OK;
        };
        CORU_CUDA(cudaEventRecord(ooc_ev[2], st));  // both buffers start free (main-stream order)
        CORU_CUDA(cudaEventRecord(ooc_ev[3], st));
        CORU_TRY(issue(0));
        for (int64_t i = 0; i < nch; ++i) {
            if (i + 1 < nch) CORU_TRY(issue(i + 1));
            const int b = int(i & 1);
            CORU_CUDA(cudaStreamWaitEvent(st, ooc_ev[b], 0));
            const int64_t r0 = i * cr, rows = std::min(cr, HR - r0);
            CORU_TRY(on_chunk(i, r0, rows, static_cast<const T*>(w.cbuf[b])));
            CORU_CUDA(cudaEventRecord(ooc_ev[2 + b], st));
        }
        return CORU_OK;
    };
    if (r.a_host) {
        // Each power round reads A once: c1 rows of chunk i = A_i·c2, and the partial A_i^T·c1_i from
        // the same chunk, summed into the next c2 in chunk order (deterministic).
        CORU_CUDA(cudaMemsetAsync(w.flag + 1, 0, sizeof(int), st));
        // ULV (A' = A^T, host rows of A are columns of A'): c1 = A'·c2 = sum_i A_i^T c2_i needs the
        // whole sum before c2' = A'^T c1 = [A_i c1]_i, so a round reads A twice (partials first).
        for (int i = 0; i <= r.q && r.trans; ++i) {
            CORU_TRY(stream_a([&](int64_t ch, int64_t r0, int64_t rows, const T* Ai) -> int {
                if (i == 0) {
                    CORU_CUDA(any_nonfinite_acc<T>(Ai, rows * HL, w.flag + 1, st));
                    ++g_launches;
                }
                T* out = ch == 0 ? w.b1 : w.part;
                CORU_TRY(gemm<T>(c, Op::T, Ai, HL, w.b2 + r0 * dp, dp, out, dp, R, rows, d, w.gws, w.gws_elems));
                if (ch > 0) {
                    CORU_CUDA(add_inplace<T>(w.b1, w.part, size_t(R) * dp, st));
                    ++g_launches;
                }
                return CORU_OK;
            }));
            if (i == 0) {
                int bad = 0;
                CORU_CUDA(cudaMemcpyAsync(&bad, w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
                CORU_CUDA(cudaStreamSynchronize(st));
                if (bad) return fail(CORU_EINVAL, "Matrix: non-finite entry");
            }
            if (i == r.q && w.b2prev)
                CORU_CUDA(cudaMemcpyAsync(w.b2prev, w.b2, size_t(N) * dp * sizeof(T), cudaMemcpyDeviceToDevice, st));
            CORU_TRY(stream_a([&](int64_t, int64_t r0, int64_t rows, const T* Ai) -> int {
                return gemm<T>(c, Op::N, Ai, HL, w.b1, dp, w.b2n + r0 * dp, dp, rows, R, d, w.gws, w.gws_elems);
            }));
            std::swap(w.b2, w.b2n);
        }
        for (int i = 0; i <= r.q && !r.trans; ++i) {
            CORU_TRY(stream_a([&](int64_t ch, int64_t r0, int64_t rows, const T* Ai) -> int {
                if (i == 0) {  // finiteness, as the Matrix constructor / read_matrix_bin (matrix.hpp:29-31)
                    CORU_CUDA(any_nonfinite_acc<T>(Ai, rows * N, w.flag + 1, st));
                    ++g_launches;
                }
                CORU_TRY(gemm<T>(c, Op::N, Ai, N, w.b2, dp, w.b1 + r0 * dp, dp, rows, N, d, w.gws, w.gws_elems));
                T* out = ch == 0 ? w.b2n : w.part;
                CORU_TRY(gemm<T>(c, Op::T, Ai, N, w.b1 + r0 * dp, dp, out, dp, N, rows, d, w.gws, w.gws_elems));
                if (ch > 0) {
                    CORU_CUDA(add_inplace<T>(w.b2n, w.part, size_t(N) * dp, st));
                    ++g_launches;
                }
                return CORU_OK;
            }));
            if (i == 0) {
                int bad = 0;
                CORU_CUDA(cudaMemcpyAsync(&bad, w.flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
                CORU_CUDA(cudaStreamSynchronize(st));
                if (bad) return fail(CORU_EINVAL, "Matrix: non-finite entry");
            }
            if (i == r.q && w.b2prev)
                CORU_CUDA(cudaMemcpyAsync(w.b2prev, w.b2, size_t(N) * dp * sizeof(T), cudaMemcpyDeviceToDevice, st));
            std::swap(w.b2, w.b2n);
        }
    }
    for (int i = r.first_done ? 1 : 0; i <= r.q && !r.a_host; ++i) {
        if (!(i == 0 && sketch_done))
            CORU_TRY(gemm<T>(c, r.op_a(), r.A, r.lda, w.b2, dp, w.b1, dp, R, N, d, w.gws, w.gws_elems));
        if (i == r.q && early_qr1) {
            CORU_CUDA(cudaEventRecord(c->ev_fork, st));
            CORU_CUDA(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
            CORU_TRY(w.ts1.factor(w.b1, dp, w.r1, c->aux));  // Q1, R1 = QR(c1) (corutv.hpp:59)
            CORU_TRY(w.ts1.form_q(nullptr, w.q1, dp, c->aux));
            CORU_CUDA(conditioning_flag<T>(w.r1, d, d, w.flag, c->aux));  // corutv.hpp:61-64
            ++g_launches;
        }
        if (i == r.q && w.b2prev)
            CORU_CUDA(cudaMemcpyAsync(w.b2prev, w.b2, size_t(N) * dp * sizeof(T), cudaMemcpyDeviceToDevice, st));
        c->prof_overlap = i == r.q && early_qr1;  // the Q1 tree runs on the aux stream under this pass
        if (w.b2chunks) {
            // per-chunk product -> contiguous chunk buffer -> all-reduce + scatter on the aux stream,
            // overlapping the next chunk's product on the main stream
            int64_t off = 0;
            for (int c0 = 0; c0 < d; c0 += kB2ChunkCols) {
                const int nc = std::min(kB2ChunkCols, d - c0);
                const int ncp = int(round_up(nc, 8));
                T* chunk = w.b2chunks + off;
                CORU_TRY(gemm<T>(c, r.op_at(), r.A, r.lda, w.b1 + c0, dp, chunk, ncp, N, R, nc, w.gws, w.gws_elems));
                CORU_CUDA(cudaEventRecord(c->ev_fork, st));
                CORU_CUDA(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
                CORU_TRY(allreduce<T>(c, chunk, size_t(N) * ncp, c->aux));
                CORU_CUDA(copy_block<T>(chunk, ncp, w.b2 + c0, dp, N, nc, c->aux));
                ++g_launches;
                off += N * int64_t(ncp);
            }
            CORU_CUDA(cudaEventRecord(c->ev_join, c->aux));
            CORU_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
        } else {
            CORU_TRY(gemm<T>(c, r.op_at(), r.A, r.lda, w.b1, dp, w.b2, dp, N, R, d, w.gws, w.gws_elems));
            CORU_TRY(allreduce<T>(c, w.b2, size_t(N) * dp));
        }
        c->prof_overlap = false;
    }
    if (sharded) {
        // Q2 = QR(c2) (corutv.hpp:60): c2 is replicated, every rank computes the same tree (aux).
        CORU_CUDA(cudaEventRecord(c->ev_fork, st));
        CORU_CUDA(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
        CORU_TRY(w.ts2.factor(w.b2, dp, w.r2, c->aux));
        CORU_TRY(w.ts2.form_q(nullptr, w.q2, dp, c->aux));
        // Q1, R1 (main stream). Wide sketches: CholeskyQR2 over all ranks — the two Gram matrices are
        // all-reduced (d x d, identical bytes everywhere, so R1, the status and every rank's solve
        // agree), Q1_g = c1_g R^{-1} is local. Then the Householder path, which for wide sketches
        // runs only if that status says ill-conditioned (device-side gate, no host decision): local
        // tree, all-gather of the R_g, redundant top level, local Q.
        if (w.ts1.chol) {
            const CholQrReduce red = [&](double* buf, size_t count) -> cudaError_t {
                return allreduce<double>(c, buf, count) == CORU_OK ? cudaSuccess : cudaErrorUnknown;
            };
            CORU_TRY(w.ts1.factor_chol(w.b1, dp, w.r1, st, &red));
            CORU_TRY(w.ts1.form_q_chol(w.q1, dp, st));
        }
        CORU_TRY(w.ts1.factor_tree(w.b1, dp, w.r1loc, st));
        CORU_TRY(allgather<T>(c, w.r1loc, w.rstack, size_t(d) * d));
        CORU_TRY(w.tstop.factor(w.rstack, d, w.r1, st));
        CORU_TRY(w.tstop.form_q(nullptr, w.qtop, d, st));
        CORU_TRY(w.ts1.form_q_tree(w.qtop + int64_t(c->rank) * d * d, w.q1, dp, st));
        CORU_CUDA(conditioning_flag<T>(w.r1, d, d, w.flag, st));
        ++g_launches;
    } else {
        if (!early_qr1) {
            // QR(c1) on the aux stream, concurrent with QR(c2): both trees start once the last
            // A^T pass is done (overlapping that pass only slows it; QR(c2) is the critical path)
            CORU_CUDA(cudaEventRecord(c->ev_fork, st));
            CORU_CUDA(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
            CORU_TRY(w.ts1.factor(w.b1, dp, w.r1, c->aux));  // Q1, R1 = QR(c1) (corutv.hpp:59)
            CORU_TRY(w.ts1.form_q(nullptr, w.q1, dp, c->aux));
            CORU_CUDA(conditioning_flag<T>(w.r1, d, d, w.flag, c->aux));  // corutv.hpp:61-64
            ++g_launches;
        }
        CORU_TRY(w.ts2.factor(w.b2, dp, w.r2, st));  // Q2 = QR(c2) (corutv.hpp:60)
        CORU_TRY(w.ts2.form_q(nullptr, w.q2, dp, st));
    }
    CORU_CUDA(cudaEventRecord(c->ev_join, c->aux));
    // exact-D, single GPU: the projection pass W = A·Q2 needs only Q2 (main stream), so it starts
    // while the Q1 tree may still be finishing on the aux stream; the join moves after it.
    const bool late_join = w.wproj != nullptr;  // W gets its own buffer: the Q1 tree may still read c1
    if (!late_join) CORU_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));

    if (r.mode == Mode::Sketch) {
        CORU_CUDA(copy_block<T>(w.q1, dp, r.q1, r.ldq1, R, d, st));
        CORU_CUDA(copy_block<T>(w.q2, dp, r.q2, r.ldq2, N, d, st));
        g_launches += 2;
        if (r.c1) {
            CORU_CUDA(copy_block<T>(w.b1, dp, r.c1, r.ldc1, R, d, st));
            ++g_launches;
        }
        if (r.c2p) {
            CORU_CUDA(copy_block<T>(w.b2prev, dp, r.c2p, r.ldc2, N, d, st));
            ++g_launches;
        }
        int flag = 0;
        CORU_CUDA(cudaMemcpyAsync(&flag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaStreamSynchronize(st));
        if (r.warn_host) *r.warn_host = flag;
        return CORU_OK;
    }

    if (r.variant == CORU_D_APPROX) {
        // D = (Q1^T c1)·pinv(Q2^T c2_prev) (corutv.hpp:91-92): no further pass over A. Q1^T c1 is
        // summed over ranks; Q2, c2_prev and so the pinv are replicated (identical bytes).
        const bool p = c->prof;
        c->prof = false;
        int rc = gemm_tn_core<T>(c, w.q1, dp, w.b1, dp, R, d, w.y1, dp, w.tnp, w.gws, w.gws_elems);
        if (rc == CORU_OK) rc = allreduce<T>(c, w.y1, size_t(d) * dp);
        if (rc == CORU_OK) rc = gemm_tn_core<T>(c, w.q2, dp, w.b2prev, dp, N, d, w.y2, dp, w.tnp, w.gws, w.gws_elems);
        if (rc == CORU_OK) {
            const cudaError_t e = pinv_square<T>(w.y2, dp, d, w.pinv, dp, w.pws, nullptr, c->max_smem, st);
            if (e != cudaSuccess) rc = fail(CORU_ECUDA, std::string("pinv_square: ") + cudaGetErrorString(e));
            g_launches += kPinvLaunches;
        }
        if (rc == CORU_OK) rc = gemm<T>(c, Op::N, w.y1, dp, w.pinv, dp, w.m, dp, d, d, d, w.gws, w.gws_elems);
        c->prof = p;
        CORU_TRY(rc);
    } else {
        // D = (Q1^T a) q2 (corutv.hpp:90) as Q1^T (A'·Q2): W = A'·Q2 reuses the B1 buffer.
        T* W = w.wproj ? w.wproj : w.b1;
        if (r.a_host && r.trans)  // W = A'·Q2 = sum_i A_i^T Q2_i, chunk-ordered partial sums
            CORU_TRY(stream_a([&](int64_t ch, int64_t r0, int64_t rows, const T* Ai) -> int {
                T* out = ch == 0 ? W : w.part;
                CORU_TRY(gemm<T>(c, Op::T, Ai, HL, w.q2 + r0 * dp, dp, out, dp, R, rows, d, w.gws, w.gws_elems));
                if (ch > 0) {
                    CORU_CUDA(add_inplace<T>(W, w.part, size_t(R) * dp, st));
                    ++g_launches;
                }
                return CORU_OK;
            }));
        else if (r.a_host)
            CORU_TRY(stream_a([&](int64_t, int64_t r0, int64_t rows, const T* Ai) -> int {
                return gemm<T>(c, Op::N, Ai, N, w.q2, dp, W + r0 * dp, dp, rows, N, d, w.gws, w.gws_elems);
            }));
        else {
            c->prof_overlap = late_join;  // the Q1 tree may still be running on the aux stream
            const int rc = gemm<T>(c, r.op_a(), r.A, r.lda, w.q2, dp, W, dp, R, N, d, w.gws, w.gws_elems);
            c->prof_overlap = false;
            CORU_TRY(rc);
        }
        if (late_join) CORU_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));  // Q1 (and the flag) from here on
        const bool p = c->prof;  // Q1^T·W is m x d x d, not an A-pass
        c->prof = false;
        const int rc = gemm_tn_core<T>(c, w.q1, dp, W, dp, R, d, w.m, dp, w.tnp, w.gws, w.gws_elems);
        c->prof = p;
        CORU_TRY(rc);
        CORU_TRY(allreduce<T>(c, w.m, size_t(d) * dp));
    }

    // QRCP of the core (corutv.hpp:93), then the lift (corutv.hpp:94-97).
    CORU_CUDA(cudaMemsetAsync(w.qm, 0, size_t(dp) * dp * sizeof(T), st));
    CORU_CUDA(qrcp<T>(w.m, dp, d, w.qm, dp, w.tm, d, w.perm, w.qrcp_scr, c->max_smem, st));
    ++g_launches;
    {
        const bool p = c->prof;  // U = Q1·Q_M is m x d x d, not an A-pass
        c->prof = false;
        const int rc = gemm<T>(c, Op::N, w.q1, dp, w.qm, dp, r.u, r.ldu, R, d, d, w.gws, w.gws_elems);
        c->prof = p;
        CORU_TRY(rc);
    }
    CORU_CUDA(gather_columns<T>(w.q2, dp, w.perm, N, d, r.v, r.ldv, st));
    ++g_launches;
    if (r.t_transpose) CORU_CUDA(transpose_square<T>(w.tm, d, r.t, int(r.ldt), d, st));
    else CORU_CUDA(copy_block<T>(w.tm, d, r.t, r.ldt, d, d, st));
    ++g_launches;

    if (r.capture) {
        CORU_CUDA(cudaMemcpyAsync(c->host_out, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        if (r.perm_host)
            CORU_CUDA(cudaMemcpyAsync(c->host_out + 1, w.perm, sizeof(int64_t) * d, cudaMemcpyDeviceToHost, st));
        return CORU_OK;
    }
    int flag = 0;
    CORU_CUDA(cudaMemcpyAsync(&flag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (r.perm_host) CORU_CUDA(cudaMemcpyAsync(r.perm_host, w.perm, sizeof(int64_t) * d, cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    if (r.warn_host) *r.warn_host = flag;
    return CORU_OK;
}

// Small in-core single-GPU decompositions are launch-bound (C1: ~25 kernels of a few microseconds
// each, two streams): the second call with the same buffers and parameters captures the whole
// enqueue of run_impl into a CUDA graph, later calls replay it. Per call the host still generates
// the reference Φ (the seed is not part of the key) into the pinned buffer the graph uploads from.
// The kernels and their order are those of the plain path, so the results are bit-identical.
constexpr int kGraphMaxEntries = 8;
template <typename T>
bool graph_eligible(const coru_ctx* c, const Request<T>& r) {
    static const bool off = getenv("CORU_NO_GRAPH") != nullptr && atoi(getenv("CORU_NO_GRAPH")) != 0;
    if (off || c->world > 1 || c->comm || c->tcomm || c->prof || r.a_host || r.mode != Mode::Full) return false;
    if (c->stream == nullptr || c->stream == cudaStreamLegacy) return false;  // the legacy stream cannot be captured
    if (c->phi_mode != CORU_PHI_HOST_EXACT || r.d > 112) return false;   // wider cores use cooperative grids
    if (std::is_same<T, double>::value && c->f64_engine != CORU_F64_AUTO) return false;
    return r.rows * r.cols <= (int64_t(1) << 24);
}

template <typename T>
int run_graph(coru_ctx* c, const Request<T>& r0) {
    Request<T> r = r0;
    const int d = r.d, dp = int(round_up(d, 8));
    const int64_t N = r.cols;
    coru_ctx::GraphEntry* e = nullptr;
    for (auto& g : c->graphs)
        if (g.A == r.A && g.lda == r.lda && g.rows == r.rows && g.cols == r.cols && g.d == d && g.q == r.q &&
            g.variant == r.variant && g.elem == int(sizeof(T)) && g.trans == r.trans && g.u == r.u && g.t == r.t &&
            g.v == r.v && g.ldu == r.ldu && g.ldt == r.ldt && g.ldv == r.ldv && g.want_perm == (r.perm_host != nullptr) &&
            g.stream == c->stream)
            e = &g;
    if (!e) {  // first sighting: run the plain path (it also sizes the arena and sets every kernel attribute)
        if (int(c->graphs.size()) >= kGraphMaxEntries) {
            size_t lru = 0;
            for (size_t i = 1; i < c->graphs.size(); ++i)
                if (c->graphs[i].last_use < c->graphs[lru].last_use) lru = i;
            if (c->graphs[lru].exec) cudaGraphExecDestroy(c->graphs[lru].exec);
            c->graphs.erase(c->graphs.begin() + long(lru));
        }
        coru_ctx::GraphEntry g;
        g.A = r.A; g.lda = r.lda; g.rows = r.rows; g.cols = r.cols; g.d = d; g.q = r.q; g.variant = r.variant;
        g.elem = int(sizeof(T)); g.trans = r.trans; g.u = r.u; g.t = r.t; g.v = r.v; g.ldu = r.ldu; g.ldt = r.ldt;
        g.ldv = r.ldv; g.want_perm = r.perm_host != nullptr; g.stream = c->stream; g.last_use = ++c->graph_clock;
        c->graphs.push_back(g);
        return run<T>(c, r);
    }
    e->last_use = ++c->graph_clock;
    if (e->state < 0) return run<T>(c, r);
    if (e->state == 1 && (e->arena != c->arena || e->pinned != c->pinned)) {  // buffers moved: capture again
        cudaGraphExecDestroy(e->exec);
        e->exec = nullptr;
        e->state = 0;
    }
    if (!c->host_out && cudaMallocHost(reinterpret_cast<void**>(&c->host_out), sizeof(int64_t) * 160) != cudaSuccess) {
        cudaGetLastError();
        c->host_out = nullptr;
        return run<T>(c, r);
    }
    // Φ for this call: the reference's gaussian(cols, ell, {seed, stream}), padded to dp, in the pinned buffer
    CORU_TRY(ensure_pinned(c, size_t(N) * dp * sizeof(T)));
    CORU_CUDA(cudaEventSynchronize(c->ev_phi));
    gaussian_host_rows<T>(N, d, r.seed, r.stream, reinterpret_cast<T*>(c->pinned), dp, c->host_threads, 1, 0, N);
    c->oz_a = nullptr;
    c->last_f64_engine = 0;
    if (e->state == 0) {
        const void* pinned_before = c->pinned;
        r.capture = true;
        const int64_t l0 = g_launches;
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            e->state = -1;
            return run<T>(c, r0);
        }
        const int rc = run_impl<T>(c, r, 0);
        const cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
        cudaError_t ie = cudaSuccess;
        if (rc != CORU_OK || ce != cudaSuccess || !graph ||
            (ie = cudaGraphInstantiate(&e->exec, graph, 0)) != cudaSuccess) {
            if (getenv("CORU_GRAPH_DEBUG"))
                fprintf(stderr, "coru: graph capture failed: rc %d (%s), end-capture %s, instantiate %s\n", rc,
                        g_err.c_str(), cudaGetErrorString(ce), cudaGetErrorString(ie));
            cudaGetLastError();
            if (graph) cudaGraphDestroy(graph);
            e->exec = nullptr;
            e->state = -1;
            g_launches = l0;
            return run<T>(c, r0);
        }
        cudaGraphDestroy(graph);
        e->launches = g_launches - l0;
        g_launches = l0;
        e->arena = c->arena;
        e->pinned = pinned_before;
        e->state = 1;
    }
    CORU_CUDA(cudaGraphLaunch(e->exec, c->stream));
    g_launches += e->launches;
    ++c->graph_replays;
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    if (r.warn_host) *r.warn_host = int(reinterpret_cast<int*>(c->host_out)[0]);
    if (r.perm_host) std::memcpy(r.perm_host, c->host_out + 1, sizeof(int64_t) * size_t(d));
    return CORU_OK;
}

int enter(coru_ctx* c) {
    if (!c) return fail(CORU_EINVAL, "null context");
    CORU_CUDA(cudaSetDevice(c->device));
    return CORU_OK;
}

template <typename T>
int corutv_dev(coru_ctx* c, const T* A, int64_t m_local, int64_t m, int64_t n, int64_t lda, int64_t ell, int q,
               int variant, uint64_t seed, uint64_t stream, coru_utv* out) {
    CORU_TRY(check_params(m, n, ell, q));
    if (variant != CORU_D_EXACT && variant != CORU_D_APPROX) return fail(CORU_EINVAL, "corutv: unknown DVariant");
    if (!out || !A) return fail(CORU_EINVAL, "null argument");
    if (c->world <= 1 && m_local != m) return fail(CORU_EINVAL, "m_local != m without a communicator");
    if (lda < n) return fail(CORU_EINVAL, "lda < n");
    Request<T> r;
    r.A = A;
    r.lda = lda;
    r.d = int(ell);
    r.q = q;
    r.seed = seed;
    r.stream = stream;
    r.variant = variant;
    r.perm_host = out->perm;
    r.warn_host = &out->conditioning_warning;
    if (m < n) {
        if (c->world > 1) return fail(CORU_ENOTSUP, "row-sharded ULV (rows < cols) is not supported");
        // corutv(a^T) then {v, t^T, u, lower = true} (corutv.hpp:82-87).
        r.trans = true;
        r.rows = n;
        r.cols = m;
        r.u = static_cast<T*>(out->v);
        r.ldu = out->ldv;
        r.v = static_cast<T*>(out->u);
        r.ldv = out->ldu;
        r.t = static_cast<T*>(out->t);
        r.ldt = out->ldt;
        r.t_transpose = true;
        out->lower = 1;
    } else {
        r.rows = m_local;
        r.cols = n;
        r.u = static_cast<T*>(out->u);
        r.ldu = out->ldu;
        r.v = static_cast<T*>(out->v);
        r.ldv = out->ldv;
        r.t = static_cast<T*>(out->t);
        r.ldt = out->ldt;
        out->lower = 0;
    }
    if (graph_eligible<T>(c, r)) return run_graph<T>(c, r);
    return run<T>(c, r);
}

// Out-of-core corutv (§8 f4): A in host memory, streamed. Unregistered host memory is page-locked
// (read-only) for the duration of the call so every stream runs at full link bandwidth.
template <typename T>
int corutv_ooc(coru_ctx* c, const T* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q, int variant,
               uint64_t seed, uint64_t stream, int64_t chunk_rows, coru_utv* out) {
    CORU_TRY(check_params(m, n, ell, q));
    if (variant != CORU_D_EXACT && variant != CORU_D_APPROX) return fail(CORU_EINVAL, "corutv: unknown DVariant");
    if (!out || !A) return fail(CORU_EINVAL, "null argument");
    if (lda < n) return fail(CORU_EINVAL, "lda < n");
    if (c->world > 1) return fail(CORU_EINVAL, "out-of-core corutv is single-GPU");
    if (chunk_rows <= 0) chunk_rows = std::max<int64_t>(1, int64_t((size_t(512) << 20) / (size_t(n) * sizeof(T))));
    chunk_rows = std::min(chunk_rows, m);
    const bool trans = m < n;  // corutv(a^T) then {v, t^T, u, lower = true} (corutv.hpp:82-87)
    Request<T> r;
    r.a_host = A;
    r.ooc_rows = chunk_rows;
    r.lda = lda;
    r.trans = trans;
    r.rows = trans ? n : m;
    r.cols = trans ? m : n;
    r.d = int(ell);
    r.q = q;
    r.seed = seed;
    r.stream = stream;
    r.variant = variant;
    r.perm_host = out->perm;
    r.warn_host = &out->conditioning_warning;
    r.u = static_cast<T*>(trans ? out->v : out->u);
    r.ldu = trans ? out->ldv : out->ldu;
    r.v = static_cast<T*>(trans ? out->u : out->v);
    r.ldv = trans ? out->ldu : out->ldv;
    r.t = static_cast<T*>(out->t);
    r.ldt = out->ldt;
    r.t_transpose = trans;
    out->lower = trans ? 1 : 0;
    // Host output buffers (the C++ drop-in passes coru::Matrix storage): run into device scratch
    // and copy back (U m x ell, T ell x ell, V n x ell with the caller's leading dimensions).
    auto is_host = [](const void* ptr) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
            cudaGetLastError();
            return true;
        }
        return a.type == cudaMemoryTypeUnregistered || a.type == cudaMemoryTypeHost;
    };
    T* dev_out = nullptr;
    if (is_host(out->u) || is_host(out->t) || is_host(out->v)) {
        const size_t elems = size_t(m) * ell + size_t(ell) * ell + size_t(n) * ell;
        if (cudaMalloc(&dev_out, elems * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            return fail(CORU_ENOMEM, "cudaMalloc of the out-of-core output buffers failed");
        }
        T* du = dev_out;                                          // U: m x ell
        T* dv = dev_out + size_t(m) * ell + size_t(ell) * ell;    // V: n x ell
        r.u = trans ? dv : du;
        r.ldu = ell;
        r.t = dev_out + size_t(m) * ell;
        r.ldt = ell;
        r.v = trans ? du : dv;
        r.ldv = ell;
    }
    bool registered = false;
    cudaPointerAttributes pa{};
    const size_t bytes = size_t(m - 1) * lda * sizeof(T) + size_t(n) * sizeof(T);
    if (cudaPointerGetAttributes(&pa, A) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered) {
        cudaGetLastError();
        registered = cudaHostRegister(const_cast<T*>(A), bytes, cudaHostRegisterReadOnly) == cudaSuccess;
        cudaGetLastError();  // registration is an optimisation: pageable copies still work
    }
    int rc = run<T>(c, r);
    if (dev_out) {
        if (rc == CORU_OK) {
            auto back = [&](void* dst, int64_t ldd, const T* src, int64_t rows) -> cudaError_t {
                return cudaMemcpy2DAsync(dst, size_t(ldd) * sizeof(T), src, size_t(ell) * sizeof(T),
                                         size_t(ell) * sizeof(T), size_t(rows), cudaMemcpyDeviceToHost, c->stream);
            };
            const T* du = dev_out;
            const T* dv = dev_out + size_t(m) * ell + size_t(ell) * ell;
            cudaError_t e = back(out->u, out->ldu, du, m);
            if (e == cudaSuccess) e = back(out->t, out->ldt, r.t, ell);
            if (e == cudaSuccess) e = back(out->v, out->ldv, dv, n);
            if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
            if (e != cudaSuccess) rc = fail(CORU_ECUDA, std::string("output copy: ") + cudaGetErrorString(e));
        }
        cudaStreamSynchronize(c->stream);
        cudaFree(dev_out);
    }
    if (registered) {
        cudaStreamSynchronize(c->stream);
        cudaStreamSynchronize(c->aux);
        cudaHostUnregister(const_cast<T*>(A));
    }
    return rc;
}

template <typename T>
__global__ void k_sum_chunks(const T* __restrict__ parts, int nparts, int64_t rows, int d, int ldp, int64_t stride,
                             T* __restrict__ out, int ldo) {
    const int64_t total = rows * d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / d;
        const int cc = int(e - r * d);
        T s = parts[r * ldp + cc];
        for (int i = 1; i < nparts; ++i) s += parts[i * stride + r * ldp + cc];  // fixed chunk order
        out[r * ldo + cc] = s;
    }
}
template <typename T>
cudaError_t sum_chunks(const T* parts, int nparts, int64_t rows, int d, int ldp, int64_t stride, T* out, int ldo,
                       cudaStream_t st) {
    const int blocks = int(std::min<int64_t>((rows * d + 255) / 256, 148 * 8));
    k_sum_chunks<T><<<std::max(blocks, 1), 256, 0, st>>>(parts, nparts, rows, d, ldp, stride, out, ldo);
    return cudaGetLastError();
}

// Host-buffer entry: upload A into the arena head, run, download. Single GPU.
template <typename T>
int corutv_host(coru_ctx* c, const T* A, int64_t m, int64_t n, int64_t ell, int q, int variant, uint64_t seed,
                uint64_t stream, T* U, T* Tt, T* V, int64_t* perm, int* lower, int* warn) {
    CORU_TRY(check_params(m, n, ell, q));
    if (variant != CORU_D_EXACT && variant != CORU_D_APPROX) return fail(CORU_EINVAL, "corutv: unknown DVariant");
    if (!A || !U || !Tt || !V) return fail(CORU_EINVAL, "null argument");
    if (c->world > 1) return fail(CORU_EINVAL, "host-buffer entry is single-GPU; use the _dev entry per rank");
    c->oz_pre_a = nullptr;  // nothing pre-computed yet for this call's A
    const bool trans = m < n;
    const int d = int(ell), dp = int(round_up(ell, 8));
    // Upload pipeline (m >= n, A of 32 MB and more): A arrives in row chunks on the aux stream while
    // the main stream validates each chunk and runs the first power round on it (c1 rows = A_i·Φ,
    // partial c2 = A_i^T·c1_i, summed in chunk order), so the first two passes and the finiteness
    // check hide under the H2D copy. Later rounds need all of A and start after the last chunk.
    constexpr int C = coru_ctx::kUploadChunks;
    const bool pipe = !trans && m >= int64_t(C) * 2 * (ell + 1) && size_t(m) * n * sizeof(T) >= (size_t(32) << 20) &&
                      getenv("CORU_NO_UPLOAD_PIPE") == nullptr;
    auto chunk_rows = [&](int i, int64_t& r0, int64_t& rows) {
        r0 = m * i / C;
        rows = m * (i + 1) / C - r0;
    };
    int64_t cwse = 0;
    if (pipe)
        for (int i = 0; i < C; ++i) {
            int64_t r0, rows;
            chunk_rows(i, r0, rows);
            cwse = std::max({cwse, gemm_ws<T>(Op::N, rows, n, d, c->num_sms), gemm_ws<T>(Op::T, n, rows, d, c->num_sms)});
        }
    // Head of the arena: A, U, T, V and a flag (+ the pipeline's partial sketches and GEMM
    // workspace), then the decomposition workspace.
    Carver head{nullptr, 0};
    T* parts = nullptr;
    T* cws = nullptr;
    auto lay = [&](Carver& cv, T*& a, T*& u, T*& t, T*& v, int*& f) {
        a = cv.template take<T>(m * n);
        u = cv.template take<T>(m * ell);
        t = cv.template take<T>(ell * ell);
        v = cv.template take<T>(n * ell);
        f = cv.template take<int>(4);
        if (pipe) {
            parts = cv.template take<T>(int64_t(C) * n * dp);
            cws = cv.template take<T>(cwse);
        }
    };
    T *a_d, *u_d, *t_d, *v_d;
    int* f_d;
    lay(head, a_d, u_d, t_d, v_d, f_d);
    const size_t head_bytes = (head.off + 255) / 256 * 256;
    coru_utv out{nullptr, ell, nullptr, ell, nullptr, ell, perm, 0, 0};
    Request<T> r;
    r.lda = n;
    r.d = d;
    r.q = q;
    r.seed = seed;
    r.stream = stream;
    r.variant = variant;
    r.perm_host = perm;
    r.warn_host = &out.conditioning_warning;
    r.rows = trans ? n : m;
    r.cols = trans ? m : n;
    r.trans = trans;
    r.t_transpose = trans;
    // Reserve the head plus the workspace before anything is placed in the arena.
    {
        Work<T> w;
        Carver meas{nullptr, head_bytes};
        w.layout(meas, c, r, dp);
        CORU_TRY(ensure_arena(c, meas.off));
    }
    Carver cv{c->arena, 0};
    lay(cv, a_d, u_d, t_d, v_d, f_d);
    r.A = a_d;
    r.u = trans ? v_d : u_d;
    r.ldu = ell;
    r.v = trans ? u_d : v_d;
    r.ldv = ell;
    r.t = t_d;
    r.ldt = ell;
    cudaStream_t st = c->stream;
    if (pipe) {
        Work<T> w;  // the exact carving run() will use
        Carver wc{c->arena, head_bytes};
        w.layout(wc, c, r, dp);
        CORU_TRY(gen_phi<T>(c, r, w.b2, dp));
        CORU_CUDA(cudaMemsetAsync(f_d, 0, sizeof(int), st));
        CORU_CUDA(cudaEventRecord(c->ev_fork, st));  // the copies may overwrite the arena from here on
        CORU_CUDA(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
        const bool prof = c->prof;  // partial passes: not A-pass launches
        c->prof = false;
        int rc = CORU_OK;
        // fp64 on the Ozaki engine: its exponent pass over A (0.7 ms at C3) runs chunk by chunk under
        // the upload as well; run() finds the exponents in place (oz_prepare)
        bool pre_exp = false;
        if constexpr (std::is_same<T, double>::value) {
            if (oz_wanted(c, m, n, d)) {
                CORU_TRY(oz_ensure_exponents(c, m, n));
                CORU_CUDA(gemm_oz_exponents_begin(m, n, c->oz_e, c->oz_e + m, st));
                pre_exp = true;
            }
        }
        for (int i = 0; i < C && rc == CORU_OK; ++i) {
            int64_t r0, rows;
            chunk_rows(i, r0, rows);
            // chunk i's H2D (staged when A is pageable) is enqueued before its GEMMs, so the host
            // copies chunk i+1 while the GPU works on chunk i
            rc = h2d(c, a_d + r0 * n, A + r0 * n, sizeof(T) * rows * n, c->aux);
            if (rc == CORU_OK && cudaEventRecord(c->ev_chunk[i], c->aux) != cudaSuccess)
                rc = fail(CORU_ECUDA, "cudaEventRecord failed");
            if (rc != CORU_OK) break;
            const T* ai = a_d + r0 * n;
            if (cudaStreamWaitEvent(st, c->ev_chunk[i], 0) != cudaSuccess ||
                any_nonfinite_acc<T>(ai, rows * n, f_d, st) != cudaSuccess) {
                rc = fail(CORU_ECUDA, "upload pipeline launch failed");
                break;
            }
            ++g_launches;
            if constexpr (std::is_same<T, double>::value) {
                if (pre_exp && gemm_oz_exponents_rows(a_d, n, r0, rows, n, c->oz_e, c->oz_e + m, st) != cudaSuccess) {
                    rc = fail(CORU_ECUDA, "upload pipeline launch failed");
                    break;
                }
            }
            rc = gemm<T>(c, Op::N, ai, n, w.b2, dp, w.b1 + r0 * dp, dp, rows, n, d, cws, cwse);  // c1 rows
            if (rc == CORU_OK)
                rc = gemm<T>(c, Op::T, ai, n, w.b1 + r0 * dp, dp, parts + int64_t(i) * n * dp, dp, n, rows, d, cws, cwse);
        }
        c->prof = prof;
        CORU_TRY(rc);
        if constexpr (std::is_same<T, double>::value) {
            if (pre_exp) {
                CORU_CUDA(gemm_oz_exponents_end(m, n, c->oz_e, c->oz_e + m, st));
                g_launches += 2 + C;
                c->oz_pre_a = a_d;
                c->oz_pre_lda = n;
                c->oz_pre_rows = m;
                c->oz_pre_cols = n;
            }
        }
        if (q == 0 && w.b2prev)  // c2_prev = Φ for the approx core (corutv.hpp:56)
            CORU_CUDA(cudaMemcpyAsync(w.b2prev, w.b2, sizeof(T) * n * dp, cudaMemcpyDeviceToDevice, st));
        CORU_CUDA(sum_chunks<T>(parts, C, n, d, dp, int64_t(n) * dp, w.b2, dp, st));  // c2 = a^T·c1, chunk order
        ++g_launches;
        r.first_done = true;
    } else {
        CORU_TRY(h2d(c, a_d, A, sizeof(T) * m * n, st));
        CORU_CUDA(any_nonfinite<T>(a_d, m * n, f_d, st));
        ++g_launches;
    }
    {
        // The Matrix constructor rejects non-finite entries (matrix.hpp:29-31); no output is written.
        int bad = 0;
        CORU_CUDA(cudaMemcpyAsync(&bad, f_d, sizeof(int), cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaStreamSynchronize(st));
        if (bad) return fail(CORU_EINVAL, "Matrix: non-finite entry");
    }
    CORU_TRY(run<T>(c, r, head_bytes));
    CORU_TRY(d2h_sync(c, U, u_d, sizeof(T) * m * ell, st));
    CORU_TRY(d2h_sync(c, Tt, t_d, sizeof(T) * ell * ell, st));
    CORU_TRY(d2h_sync(c, V, v_d, sizeof(T) * n * ell, st));
    if (lower) *lower = m < n ? 1 : 0;
    if (warn) *warn = out.conditioning_warning;
    return CORU_OK;
}


// ==== SVD-based baselines (baselines.hpp:43-71), fp64 =========================================
__global__ void k_transpose_rect(const double* __restrict__ src, int64_t lds, int64_t rows, int cols,
                                 double* __restrict__ dst, int64_t ldd) {
    // dst (cols x rows) = src (rows x cols)^T
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e / rows);
        const int64_t r = e - int64_t(c) * rows;
        dst[int64_t(c) * ldd + r] = src[r * lds + c];
    }
}

// Φ = gaussian(rows, d, {seed, stream}) into out (ld dp, zero padding), per the context's Φ mode.
int fill_phi(coru_ctx* c, int64_t rows, int d, int dp, uint64_t seed, uint64_t stream, double* out) {
    if (c->phi_mode == CORU_PHI_DEVICE) {
        uint64_t s4[4];
        seed_state_words(seed, stream, s4);
        CORU_CUDA(gaussian_dev<double>(rows, d, s4, out, dp, c->stream));
        ++g_launches;
        return CORU_OK;
    }
    return upload_phi_host<double>(c, rows, d, dp, seed, stream, out, c->stream);
}

// tsr_svd (baselines.hpp:43-56): two sketches (A·Φ1, A^T·Φ2), their QRs (two streams), the core
// (Q1^T Y1)·pinv(Q2^T Φ1), its Jacobi SVD, the lift. Device A, U (m x ell), V (n x ell), S (ell).
int tsr_impl(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int d, uint64_t seed, uint64_t stream,
             double* U, int64_t ldu, double* S, double* V, int64_t ldv, int* conv_host, size_t off,
             size_t* need = nullptr) {
    const int dp = int(round_up(d, 8));
    const int sms = c->num_sms;
    struct Lay {
        double *phi1, *phi2, *y1, *y2, *q1, *q2, *gws, *r1, *r2, *t1, *t2, *p, *b, *bu, *bv, *sig, *pws;
        int* conv;
        int64_t gwse;
        TsqrBufs<double> ts1, ts2;
    } l;
    auto lay = [&](Carver& cv) {
        l.phi1 = cv.take<double>(n * dp);
        l.phi2 = cv.take<double>(m * dp);
        l.y1 = cv.take<double>(m * dp);
        l.y2 = cv.take<double>(n * dp);
        l.q1 = cv.take<double>(m * dp);
        l.q2 = cv.take<double>(n * dp);
        l.gwse = std::max({gemm_ws<double>(Op::N, m, n, d, sms), gemm_ws<double>(Op::T, n, m, d, sms),
                           gemm_ws<double>(Op::T, d, m, d, sms), gemm_ws<double>(Op::T, d, n, d, sms),
                           gemm_ws<double>(Op::N, m, d, d, sms), gemm_ws<double>(Op::N, n, d, d, sms),
                           gemm_ws<double>(Op::N, d, d, d, sms)});
        l.gws = cv.take<double>(l.gwse);
        l.ts1.carve(cv, m, d, c->max_smem, sms, c->wide_qr);
        l.ts2.carve(cv, n, d, c->max_smem, sms, c->wide_qr);
        l.r1 = cv.take<double>(int64_t(d) * d);
        l.r2 = cv.take<double>(int64_t(d) * d);
        l.t1 = cv.take<double>(int64_t(d) * dp);
        l.t2 = cv.take<double>(int64_t(d) * dp);
        l.p = cv.take<double>(int64_t(d) * dp);
        l.b = cv.take<double>(int64_t(d) * dp);
        l.bu = cv.take<double>(int64_t(d) * dp);
        l.bv = cv.take<double>(int64_t(d) * dp);
        l.sig = cv.take<double>(d);
        l.pws = cv.take<double>(pinv_ws_doubles(d));
        l.conv = cv.take<int>(4);
    };
    Carver meas{nullptr, off};
    lay(meas);
    if (need) {  // sizing pass: the caller reserves the arena before placing anything in it
        *need = meas.off;
        return CORU_OK;
    }
    CORU_TRY(ensure_arena(c, meas.off));
    Carver cv{c->arena, off};
    lay(cv);
    cudaStream_t st = c->stream;
    CORU_TRY(fill_phi(c, n, d, dp, seed, stream, l.phi1));      // substream(seed, 0)
    CORU_TRY(fill_phi(c, m, d, dp, seed, stream + 1, l.phi2));  // substream(seed, 1)
    CORU_CUDA(cudaMemsetAsync(l.q1, 0, size_t(m) * dp * sizeof(double), st));
    CORU_CUDA(cudaMemsetAsync(l.q2, 0, size_t(n) * dp * sizeof(double), st));
    // y1 = A·Φ1, y2 = A^T·Φ2 (A^T never formed)
    CORU_TRY(gemm<double>(c, Op::N, A, lda, l.phi1, dp, l.y1, dp, m, n, d, l.gws, l.gwse));
    CORU_TRY(gemm<double>(c, Op::T, A, lda, l.phi2, dp, l.y2, dp, n, m, d, l.gws, l.gwse));
    CORU_CUDA(cudaEventRecord(c->ev_fork, st));
    CORU_CUDA(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
    CORU_TRY(l.ts1.factor(l.y1, dp, l.r1, c->aux));
    CORU_TRY(l.ts1.form_q(nullptr, l.q1, dp, c->aux));
    CORU_TRY(l.ts2.factor(l.y2, dp, l.r2, st));
    CORU_TRY(l.ts2.form_q(nullptr, l.q2, dp, st));
    CORU_CUDA(cudaEventRecord(c->ev_join, c->aux));
    CORU_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
    const bool prof = c->prof;  // the rest are d-wide products, not A-passes
    c->prof = false;
    int rc = gemm<double>(c, Op::T, l.q1, dp, l.y1, dp, l.t1, dp, d, m, d, l.gws, l.gwse);      // Q1^T·y1
    if (rc == CORU_OK) rc = gemm<double>(c, Op::T, l.q2, dp, l.phi1, dp, l.t2, dp, d, n, d, l.gws, l.gwse);  // Q2^T·Φ1
    if (rc == CORU_OK) {
        const cudaError_t e = pinv_square<double>(l.t2, dp, d, l.p, dp, l.pws, nullptr, c->max_smem, st);
        if (e != cudaSuccess) rc = fail(CORU_ECUDA, std::string("pinv_square: ") + cudaGetErrorString(e));
        g_launches += kPinvLaunches;
    }
    if (rc == CORU_OK) rc = gemm<double>(c, Op::N, l.t1, dp, l.p, dp, l.b, dp, d, d, d, l.gws, l.gwse);
    if (rc == CORU_OK) {
        const cudaError_t e = svd_square<double>(l.b, dp, d, l.bu, dp, l.sig, l.bv, dp, l.pws, l.conv, c->max_smem, st);
        if (e != cudaSuccess) rc = fail(CORU_ECUDA, std::string("svd_square: ") + cudaGetErrorString(e));
        g_launches += kSvdLaunches;
    }
    if (rc == CORU_OK) rc = gemm<double>(c, Op::N, l.q1, dp, l.bu, dp, U, ldu, m, d, d, l.gws, l.gwse);
    if (rc == CORU_OK) rc = gemm<double>(c, Op::N, l.q2, dp, l.bv, dp, V, ldv, n, d, d, l.gws, l.gwse);
    c->prof = prof;
    CORU_TRY(rc);
    CORU_CUDA(cudaMemcpyAsync(S, l.sig, sizeof(double) * d, cudaMemcpyDeviceToDevice, st));
    int conv = 0;
    CORU_CUDA(cudaMemcpyAsync(&conv, l.conv, sizeof(int), cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    if (conv_host) *conv_host = conv > 0 ? 1 : 0;
    return CORU_OK;
}

int check_tsr(int64_t m, int64_t n, int64_t ell) {
    if (m < 1 || n < 1) return fail(CORU_EINVAL, "Matrix: dimensions must be positive");
    if (ell < 1 || ell >= std::min(m, n)) return fail(CORU_EINVAL, "tsr_svd: ell out of range");
    return CORU_OK;
}

int check_sor(int64_t m, int64_t n, int64_t k, int64_t ell, int q) {
    if (m < 1 || n < 1) return fail(CORU_EINVAL, "Matrix: dimensions must be positive");
    // m < n recurses on the transpose (baselines.hpp:63-66), which has the same min(rows, cols)
    if (ell < 1) return fail(CORU_EINVAL, "corutv: ell must be >= 1");
    if (ell >= std::min(m, n)) return fail(CORU_EINVAL, "corutv: ell must be < min(rows, cols)");
    if (k < 1 || k > ell) return fail(CORU_EINVAL, "sor_svd: requires 1 <= k <= ell");
    if (q < 0) return fail(CORU_EINVAL, "sor_svd: q must be >= 0");
    return CORU_OK;
}

// sor_svd (baselines.hpp:61-71): the CoR sketch stage, the exact core D = Q1^T A Q2, its Jacobi SVD
// truncated to rank k, lifted to the m x n output L = Q1·C·Q2^T. For m < n the reference works on
// A^T and transposes the result; here A^T is a flag and L = Q2'·C^T·Q1'^T is written directly.
int sor_impl(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int k, int d, int q, uint64_t seed,
             uint64_t stream, double* Lout, int64_t ldl, size_t off, size_t* need = nullptr) {
    const bool trans = m < n;
    const int64_t R = trans ? n : m, N = trans ? m : n;
    const int dp = int(round_up(d, 8));
    const int sms = c->num_sms;
    const Op op_a = trans ? Op::T : Op::N;
    const int64_t mX = trans ? N : R, nY = trans ? R : N;  // L = X·C·Y^T, X mX x d, Y nY x d
    struct Lay {
        double *q1, *q2, *w, *dm, *du, *dv, *sig, *core, *coret, *t, *yt, *gws, *pws;
        int* conv;
        int64_t gwse;
    } l;
    auto lay = [&](Carver& cv) {
        l.q1 = cv.take<double>(R * dp);
        l.q2 = cv.take<double>(N * dp);
        l.w = cv.take<double>(R * dp);
        l.dm = cv.take<double>(int64_t(d) * dp);
        l.du = cv.take<double>(int64_t(d) * dp);
        l.dv = cv.take<double>(int64_t(d) * dp);
        l.sig = cv.take<double>(d);
        l.core = cv.take<double>(int64_t(d) * dp);
        l.coret = cv.take<double>(int64_t(d) * dp);
        l.t = cv.take<double>(mX * dp);
        l.yt = cv.take<double>(int64_t(d) * nY);
        l.gwse = std::max({gemm_ws<double>(op_a, R, N, d, sms), gemm_ws<double>(Op::T, d, R, d, sms),
                           gemm_ws<double>(Op::N, mX, d, d, sms), gemm_ws<double>(Op::N, mX, d, int(nY), sms)});
        l.gws = cv.take<double>(l.gwse);
        l.pws = cv.take<double>(pinv_ws_doubles(d));
        l.conv = cv.take<int>(4);
    };
    Carver meas{nullptr, off};
    lay(meas);
    const size_t work_off = (meas.off + 255) / 256 * 256;
    {
        // the sketch stage carves its workspace after ours: size the arena for both up front
        Request<double> probe;
        probe.rows = R;
        probe.cols = N;
        probe.d = d;
        probe.mode = Mode::Sketch;
        Work<double> w;
        Carver wm{nullptr, work_off};
        w.layout(wm, c, probe, dp);
        if (need) {
            *need = wm.off;
            return CORU_OK;
        }
        CORU_TRY(ensure_arena(c, wm.off));
    }
    Carver cv{c->arena, off};
    lay(cv);
    Request<double> r;  // detail::sketch_bases(a, ell, q, seed) (baselines.hpp:69)
    r.A = A;
    r.lda = lda;
    r.trans = trans;
    r.rows = R;
    r.cols = N;
    r.d = d;
    r.q = q;
    r.seed = seed;
    r.stream = stream;
    r.mode = Mode::Sketch;
    r.q1 = l.q1;
    r.ldq1 = dp;
    r.q2 = l.q2;
    r.ldq2 = dp;
    int warn = 0;
    r.warn_host = &warn;
    CORU_TRY(run<double>(c, r, work_off));
    cudaStream_t st = c->stream;
    CORU_CUDA(cudaMemsetAsync(l.core, 0, size_t(d) * dp * sizeof(double), st));
    // D = (Q1^T a) q2 (baselines.hpp:70) as Q1^T (A'·Q2)
    CORU_TRY(gemm<double>(c, op_a, A, lda, l.q2, dp, l.w, dp, R, N, d, l.gws, l.gwse));
    const bool prof = c->prof;
    c->prof = false;
    int rc = gemm<double>(c, Op::T, l.q1, dp, l.w, dp, l.dm, dp, d, R, d, l.gws, l.gwse);
    if (rc == CORU_OK) {
        cudaError_t e = svd_square<double>(l.dm, dp, d, l.du, dp, l.sig, l.dv, dp, l.pws, l.conv, c->max_smem, st);
        if (e == cudaSuccess) e = svd_truncate_core<double>(l.pws, d, k, l.core, dp, st);
        if (e != cudaSuccess) rc = fail(CORU_ECUDA, std::string("svd: ") + cudaGetErrorString(e));
        g_launches += kSvdLaunches + 1;
    }
    const double* X = trans ? l.q2 : l.q1;
    const double* Y = trans ? l.q1 : l.q2;
    const double* Cm = l.core;
    if (rc == CORU_OK && trans) {
        const cudaError_t e = transpose_square<double>(l.core, dp, l.coret, dp, d, st);
        if (e != cudaSuccess) rc = fail(CORU_ECUDA, cudaGetErrorString(e));
        ++g_launches;
        Cm = l.coret;
    }
    if (rc == CORU_OK) rc = gemm<double>(c, Op::N, X, dp, Cm, dp, l.t, dp, mX, d, d, l.gws, l.gwse);
    if (rc == CORU_OK) {
        const int blocks = int(std::min<int64_t>((nY * d + 255) / 256, int64_t(sms) * 16));
        k_transpose_rect<<<std::max(blocks, 1), 256, 0, st>>>(Y, dp, nY, d, l.yt, nY);
        ++g_launches;
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(CORU_ECUDA, cudaGetErrorString(e));
    }
    if (rc == CORU_OK) rc = gemm<double>(c, Op::N, l.t, dp, l.yt, nY, Lout, ldl, mX, d, int(nY), l.gws, l.gwse);
    c->prof = prof;
    CORU_TRY(rc);
    CORU_CUDA(cudaStreamSynchronize(st));
    return CORU_OK;
}

// RpcaConfig::validate (rpca.hpp:72-77) and the inner-step switches this build provides.
int check_rpca(const coru_rpca_config* cf, int64_t m, int64_t n) {
    if (!cf) return fail(CORU_EINVAL, "null config");
    if (m < 1 || n < 1) return fail(CORU_EINVAL, "Matrix: dimensions must be positive");
    if (!(cf->rho > 1.0)) return fail(CORU_EINVAL, "RpcaConfig: rho must be > 1");
    if (!(cf->tol > 0.0)) return fail(CORU_EINVAL, "RpcaConfig: tol must be > 0");
    if (cf->max_iter < 1) return fail(CORU_EINVAL, "RpcaConfig: max_iter must be >= 1");
    if (cf->corutv_q < 0) return fail(CORU_EINVAL, "RpcaConfig: corutv_q must be >= 0");
    if (cf->inner == CORU_RPCA_SVT_EXACT)
        return fail(CORU_ENOTSUP, "alm_rpca: the svt_exact inner (full SVD of the iterate) is not provided");
    if (cf->inner != CORU_RPCA_CORUTV) return fail(CORU_EINVAL, "alm_rpca: unknown inner");
    if (cf->thresholding != CORU_COR_SOFT && cf->thresholding != CORU_COR_HARD)
        return fail(CORU_EINVAL, "alm_rpca: unknown thresholding");
    if ((cf->mu0 <= 0.0 || cf->corutv_ell == 0) && n > 1024)
        return fail(CORU_ENOTSUP, "alm_rpca: mu0 / predict_rank defaults need cols <= 1024");
    return CORU_OK;
}

// alm_rpca (rpca.hpp:95-169) with the CoR-UTV inner step, M device m x n. Iterate buffers: X (the
// inner step's input; X_1 = M exactly, so the first step reads M), Y; S is the caller's. One host
// sync per iteration (zeta, rank; the predicted ell before the sketch when corutv_ell == 0).
int rpca_impl(coru_ctx* c, const double* Min, int64_t m, int64_t n, int64_t ldm, const coru_rpca_config& cf,
              uint64_t seed, uint64_t stream, double* Lout, int64_t ldl, double* Sout, int64_t lds,
              coru_rpca_result* res, size_t off, size_t* need = nullptr) {
    const bool hard = cf.thresholding == CORU_COR_HARD;
    const bool predict = cf.corutv_ell == 0;
    const bool gram = predict || cf.mu0 <= 0.0;
    const int64_t ell_max = std::min(m, n) - 1;
    const int dmax = int(std::max<int64_t>(1, predict ? ell_max : std::min(cf.corutv_ell, std::max<int64_t>(ell_max, 1))));
    const int dpm = int(round_up(dmax, 8));
    const int sms = c->num_sms;
    const int nparts = rpca_parts(m, n, sms);
    const bool trans = hard && m < n;  // cor_threshold's corutv runs the ULV orientation on A^T
    struct Lay {
        double *x, *y, *q1, *q2, *w, *tp, *dm, *cc, *du, *dv, *sig, *pws, *gws, *parts, *scal, *g, *gpws, *gsig;
        int* ints;
        unsigned long long* cnt;
        int64_t gwse;
    } l{};
    auto lay = [&](Carver& cv) {
        l.x = cv.take<double>(m * n);
        l.y = cv.take<double>(m * n);
        l.q1 = cv.take<double>(m * dpm);  // Q1 (soft) / U (hard)
        l.q2 = cv.take<double>(n * dpm);  // Q2 (soft) / V (hard)
        l.w = cv.take<double>(m * dpm);
        l.tp = cv.take<double>(m * dpm);
        l.dm = cv.take<double>(int64_t(dpm) * dpm);  // D (soft) / T (hard)
        l.cc = cv.take<double>(int64_t(dpm) * dpm);  // svt(D) (soft) / truncated T (hard)
        l.du = cv.take<double>(int64_t(dpm) * dpm);
        l.dv = cv.take<double>(int64_t(dpm) * dpm);
        l.sig = cv.take<double>(dpm);
        l.pws = cv.take<double>(pinv_ws_doubles(dmax));
        l.gwse = 0;
        for (int d = 1; d <= dmax; d = d < dmax ? std::min(dmax, d * 2) : dmax + 1)
            l.gwse = std::max({l.gwse, gemm_ws<double>(Op::N, m, n, d, sms), gemm_ws<double>(Op::T, d, m, d, sms),
                               gemm_ws<double>(Op::N, m, d, d, sms)});
        l.gwse = std::max(l.gwse, gemm_ws<double>(Op::N, m, dmax, dmax, sms));
        if (gram) l.gwse = std::max(l.gwse, gemm_ws<double>(Op::T, n, m, int(n), sms));
        l.gws = cv.take<double>(l.gwse);
        l.parts = cv.take<double>(nparts);
        l.scal = cv.take<double>(8);
        l.ints = cv.take<int>(8);
        l.cnt = cv.take<unsigned long long>(1);
        if (gram) {
            l.g = cv.take<double>(n * n);
            l.gsig = cv.take<double>(n);
            l.gpws = cv.take<double>(pinv_ws_doubles(int(n)));
        }
    };
    Carver meas{nullptr, off};
    lay(meas);
    const size_t work_off = (meas.off + 255) / 256 * 256;
    {
        // the inner step carves its workspace after ours: size the arena for every ell it may use
        size_t top = work_off;
        for (int d = 1; d <= dmax; ++d) {
            if (!predict && d != dmax) continue;
            Request<double> probe;
            probe.rows = trans ? n : m;
            probe.cols = trans ? m : n;
            probe.trans = trans;
            probe.d = d;
            probe.mode = hard ? Mode::Full : Mode::Sketch;
            Work<double> w;
            Carver wm{nullptr, work_off};
            w.layout(wm, c, probe, int(round_up(d, 8)));
            top = std::max(top, wm.off);
        }
        if (need) {
            *need = top;
            return CORU_OK;
        }
        CORU_TRY(ensure_arena(c, top));
    }
    Carver cv{c->arena, off};
    lay(cv);
    cudaStream_t st = c->stream;
    auto cuda_ok = [&](cudaError_t e, const char* what) {
        return e == cudaSuccess ? CORU_OK : fail(CORU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    auto fro_sq = [&](const double* A, int64_t lda, double* out) -> int {  // frobenius_norm² (matrix.hpp:133-137)
        CORU_TRY(cuda_ok(sumsq_parts(A, lda, m, n, l.parts, nparts, st), "sumsq"));
        CORU_TRY(cuda_ok(sum_parts(l.parts, nparts, out, st), "sum_parts"));
        g_launches += 2;
        return CORU_OK;
    };
    // Gram-matrix norms of an m x n iterate: out[0] = ||A||_2, out[1] = ||A||_*, out[2] = ||A||_F²
    auto gram_norms_of = [&](const double* A, int64_t lda, double* h) -> int {
        const bool prof = c->prof;
        c->prof = false;
        int rc = gemm<double>(c, Op::T, A, lda, A, lda, l.g, n, n, m, int(n), l.gws, l.gwse);
        c->prof = prof;
        CORU_TRY(rc);
        CORU_TRY(cuda_ok(svd_square<double>(l.g, n, int(n), l.g, n, l.gsig, l.g, n, l.gpws, nullptr, c->max_smem, st),
                         "svd_square(gram)"));
        CORU_TRY(cuda_ok(gram_norms(l.gsig, int(n), l.scal + 4, st), "gram_norms"));
        g_launches += kSvdLaunches + 1;
        CORU_TRY(fro_sq(A, lda, l.scal + 6));
        CORU_CUDA(cudaMemcpyAsync(h, l.scal + 4, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaStreamSynchronize(st));
        return CORU_OK;
    };

    double h3[3];
    const double lambda = cf.lambda > 0.0 ? cf.lambda : 1.0 / std::sqrt(double(std::max(m, n)));
    CORU_TRY(fro_sq(Min, ldm, l.scal));
    double mfro2 = 0.0;
    CORU_CUDA(cudaMemcpyAsync(&mfro2, l.scal, sizeof(double), cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    const double m_fro = std::sqrt(mfro2);
    double mu = cf.mu0;
    if (mu <= 0.0) {
        CORU_TRY(gram_norms_of(Min, ldm, h3));
        mu = 1.25 / h3[0];
    }
    const double mu_bar = cf.mu_bar > 0.0 ? cf.mu_bar : mu * 1e7;
    CORU_CUDA(cudaMemsetAsync(l.y, 0, sizeof(double) * m * n, st));
    const double* X = Min;  // X_1 = (M - 0) + 0·inv_mu = M
    int64_t ldx = ldm;
    res->iterations = 0;
    res->converged = 0;
    res->ell_clamped = 0;
    res->rank_l = 0;
    int last_d = 1;
    int it = 0;
    while (it < cf.max_iter) {
        ++it;
        const double inv_mu = 1.0 / mu;
        int64_t ell = cf.corutv_ell;
        if (predict) {  // predict_rank(x) + 2 (rpca.hpp:45-51,122)
            CORU_TRY(gram_norms_of(X, ldx, h3));
            const double fro = std::sqrt(h3[2]);
            int64_t k = 0;
            if (fro != 0.0) {
                const double ratio = h3[1] / fro;
                const double kk = std::ceil(ratio * ratio - 1e-9);
                k = kk < 1.0 ? 1 : int64_t(kk);
            }
            ell = k + 2;
        }
        if (ell > ell_max) {
            ell = ell_max;
            res->ell_clamped = 1;
        }
        if (ell < 1) ell = 1;
        const int d = int(ell), dp = int(round_up(d, 8));
        const uint64_t it_stream = stream + uint64_t(it);  // substream(seed, it) (rpca.hpp:129)
        const double* Vb = nullptr;
        if (hard) {
            // cor_threshold(x, inv_mu, ell, q, iter_seed) (corutv.hpp:124-134)
            CORU_TRY(check_params(m, n, ell, cf.corutv_q));
            Request<double> r;
            r.A = X;
            r.lda = ldx;
            r.d = d;
            r.q = cf.corutv_q;
            r.seed = seed;
            r.stream = it_stream;
            r.variant = CORU_D_EXACT;
            int warn = 0;
            r.warn_host = &warn;
            r.trans = trans;
            r.rows = trans ? n : m;
            r.cols = trans ? m : n;
            r.u = trans ? l.q2 : l.q1;
            r.ldu = dp;
            r.v = trans ? l.q1 : l.q2;
            r.ldv = dp;
            r.t = l.dm;
            r.ldt = dp;
            r.t_transpose = trans;
            CORU_TRY(run<double>(c, r, work_off));
            if (!predict && it < cf.max_iter) CORU_TRY(phi_prefetch<double>(c, r.cols, d, dp, seed, it_stream + 1));
            CORU_TRY(cuda_ok(cor_truncate(l.dm, dp, d, inv_mu, trans ? 1 : 0, l.cc, dp, l.ints, st), "cor_truncate"));
            ++g_launches;
        } else {
            // sketch_bases(x, ell, q, iter_seed); D = (Q1^T x) Q2; svt(D, inv_mu) (rpca.hpp:135-137)
            if (ell >= std::min(m, n)) return fail(CORU_ENOTSUP, "alm_rpca: the soft inner needs min(rows, cols) >= 2");
            Request<double> r;
            r.A = X;
            r.lda = ldx;
            r.rows = m;
            r.cols = n;
            r.d = d;
            r.q = cf.corutv_q;
            r.seed = seed;
            r.stream = it_stream;
            r.mode = Mode::Sketch;
            r.q1 = l.q1;
            r.ldq1 = dp;
            r.q2 = l.q2;
            r.ldq2 = dp;
            int warn = 0;
            r.warn_host = &warn;
            CORU_TRY(run<double>(c, r, work_off));
            // Φ of the next iteration (substream(seed, it + 1), same ell) is generated on the host while
            // the GPU runs the rest of this one
            if (!predict && it < cf.max_iter) CORU_TRY(phi_prefetch<double>(c, r.cols, d, dp, seed, it_stream + 1));
            CORU_TRY(gemm<double>(c, Op::N, X, ldx, l.q2, dp, l.w, dp, m, n, d, l.gws, l.gwse));  // X·Q2 (A-pass)
            const bool prof = c->prof;
            c->prof = false;
            int rc = gemm<double>(c, Op::T, l.q1, dp, l.w, dp, l.dm, dp, d, m, d, l.gws, l.gwse);
            c->prof = prof;
            CORU_TRY(rc);
            // The preconditioned Jacobi (QRCP first) halves the sweeps on graded cores, but the RPCA core
            // (rank-ell signal, flat spectrum) gains nothing and pays the QRCP: off unless asked for.
            static const bool precond = getenv("CORU_RPCA_SVD_PRECOND") != nullptr &&
                                        atoi(getenv("CORU_RPCA_SVD_PRECOND")) != 0;
            if (precond) {
                CORU_TRY(cuda_ok(svd_factors_precond<double>(l.dm, dp, d, l.pws, c->max_smem, st), "svd_factors"));
                g_launches += 4;
            } else {
                CORU_TRY(cuda_ok(svd_square<double>(l.dm, dp, d, l.du, dp, l.sig, l.dv, dp, l.pws, nullptr, c->max_smem,
                                                    st),
                                 "svd_square"));
                g_launches += kSvdLaunches;
            }
            CORU_TRY(cuda_ok(svt_core<double>(l.pws, d, inv_mu, l.cc, dp, l.ints, st), "svt_core"));
            ++g_launches;
        }
        Vb = l.q2;  // V (hard) / Q2 (soft), n x d
        {
            // Tp = U·Tr (hard) / Q1·svt(D) (soft): L = Tp·V^T is formed inside the update kernel
            const bool prof = c->prof;
            c->prof = false;
            const int rc = gemm<double>(c, Op::N, l.q1, dp, l.cc, dp, l.tp, dp, m, d, d, l.gws, l.gwse);
            c->prof = prof;
            CORU_TRY(rc);
        }
        const double mu_next = std::min(cf.rho * mu, mu_bar);
        RpcaStep p;
        p.inv_mu = inv_mu;
        p.mu = mu;
        p.thresh = lambda * inv_mu;
        p.inv_mu_next = 1.0 / mu_next;
        cudaEvent_t ustop = nullptr;
        if (c->prof) {
            if (c->upd_used == c->upd_events.size()) {
                cudaEvent_t a, b;
                CORU_CUDA(cudaEventCreate(&a));
                CORU_CUDA(cudaEventCreate(&b));
                c->upd_events.emplace_back(a, b);
            }
            auto& ev = c->upd_events[c->upd_used++];
            CORU_CUDA(cudaEventRecord(ev.first, st));
            ustop = ev.second;
        }
        CORU_TRY(cuda_ok(rpca_lift_update(l.tp, dp, Vb, dp, d, m, n, Min, ldm, l.y, n, l.x, n, Sout, lds, nullptr, 0, p,
                                          false, l.parts, nparts, st),
                         "rpca_lift_update"));
        if (ustop) {
            CORU_CUDA(cudaEventRecord(ustop, st));
            c->upd_flops += 2.0 * double(m) * double(n) * d;
            c->upd_bytes += 40.0 * double(m) * double(n);  // read M, Y; write S, Y, X (L never written)
        }
        CORU_TRY(cuda_ok(sum_parts(l.parts, nparts, l.scal + 1, st), "sum_parts"));
        g_launches += 2;
        double zsq = 0.0;
        int rank = 0;
        CORU_CUDA(cudaMemcpyAsync(&zsq, l.scal + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaMemcpyAsync(&rank, l.ints, sizeof(int), cudaMemcpyDeviceToHost, st));
        CORU_CUDA(cudaStreamSynchronize(st));
        res->rank_l = rank;
        mu = mu_next;
        X = l.x;
        ldx = n;
        last_d = d;
        const double zeta = std::sqrt(zsq) / m_fro;
        if (res->residuals) res->residuals[it - 1] = zeta;
        if (zeta < cf.tol) {
            res->converged = 1;
            break;
        }
    }
    res->iterations = it;
    // the final L from the last step's factors (rpca.hpp:139 / :131), written once
    RpcaStep p0{};
    CORU_TRY(cuda_ok(rpca_lift_update(l.tp, int(round_up(last_d, 8)), l.q2, int(round_up(last_d, 8)), last_d, m, n,
                                      nullptr, 0, nullptr, 0, nullptr, 0, nullptr, 0, Lout, ldl, p0, true, l.parts,
                                      nparts, st),
                     "rpca_lift"));
    CORU_TRY(cuda_ok(count_nonzero(Sout, lds, m, n, l.cnt, st), "count_nonzero"));
    g_launches += 2;
    unsigned long long nz = 0;
    CORU_CUDA(cudaMemcpyAsync(&nz, l.cnt, sizeof(nz), cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    res->s_l0 = int64_t(nz);
    return CORU_OK;
}

// Upload a host matrix into the arena head (validating finiteness like the Matrix constructor).
int upload_checked(coru_ctx* c, const double* A, int64_t count, double* a_d, int* f_d) {
    cudaStream_t st = c->stream;
    CORU_CUDA(cudaMemcpyAsync(a_d, A, sizeof(double) * count, cudaMemcpyHostToDevice, st));
    CORU_CUDA(any_nonfinite<double>(a_d, count, f_d, st));
    ++g_launches;
    int bad = 0;
    CORU_CUDA(cudaMemcpyAsync(&bad, f_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    if (bad) return fail(CORU_EINVAL, "Matrix: non-finite entry");
    return CORU_OK;
}
}  // namespace

// ==== exported C-ABI =========================================================================
extern "C" {

int coru_abi_version(void) { return CORU_GPU_ABI_VERSION; }
const char* coru_last_error(void) { return g_err.c_str(); }

int64_t coru_launch_count(int reset) {
    const int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

void coru_debug_gemm_split_cap(int cap) { gemm_f64_set_split_cap(cap); }

int coru_ctx_create(int device, coru_ctx** out) {
    if (!out) return fail(CORU_EINVAL, "null out");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(CORU_ECUDA, "no CUDA device visible (coru_gpu has no CPU fallback)");
    }
    if (device < 0 || device >= n) return fail(CORU_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    CORU_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(CORU_ECUDA, std::string("device is not sm_100 (B200): ") + prop.name);
    CORU_CUDA(cudaSetDevice(device));
    auto* c = new coru_ctx;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->max_smem = int(prop.sharedMemPerBlockOptin);
    c->host_threads = int(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return fail(CORU_ECUDA, "cudaStreamCreate failed");
    }
    c->stream = c->own_stream;
    // The aux stream carries the latency-bound work that runs beside the A-passes (the Q1 tree, the
    // per-chunk all-reduces). It gets the highest stream priority: its CTAs are scheduled before the
    // pass's queued ones, so the long dependent chain of tree levels starts at once and the
    // throughput-bound pass fills in around it (C3: 13.33 -> 13.17 ms; low priority 13.30).
    // CORU_AUX_PRIORITY=default|low overrides (tooling).
    c->stage_nt = getenv("CORU_STAGE_NT") && atoi(getenv("CORU_STAGE_NT")) != 0;
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    const char* pe = getenv("CORU_AUX_PRIORITY");
    const int aux_prio = pe && std::string(pe) == "default" ? 0 : (pe && std::string(pe) == "low" ? prio_lo : prio_hi);
    if (cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, aux_prio) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_phi, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_pf, cudaEventDisableTiming) != cudaSuccess ||
        [&] {
            for (auto& e : c->ev_chunk)
                if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return true;
            return false;
        }()) {
        coru_ctx_destroy(c);
        return fail(CORU_ECUDA, "stream/event creation failed");
    }
    *out = c;
    return CORU_OK;
}

void coru_ctx_destroy(coru_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm && nccl() && nccl()->CommDestroy) nccl()->CommDestroy(c->comm);
    if (c->tscratch) cudaFree(c->tscratch);
    if (c->arena) cudaFree(c->arena);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->stage) cudaFreeHost(c->stage);
    if (c->oz_e) cudaFree(c->oz_e);
    if (c->oz_ws) cudaFree(c->oz_ws);
    if (c->oz_planes) cudaFree(c->oz_planes);
    for (auto& e : c->ev_stage)
        if (e) cudaEventDestroy(e);
    if (c->aux) {
        cudaStreamSynchronize(c->aux);
        cudaStreamDestroy(c->aux);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_phi) cudaEventDestroy(c->ev_phi);
    if (c->pf_thread.joinable()) c->pf_thread.join();
    for (auto& g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (c->host_out) cudaFreeHost(c->host_out);
    if (c->ev_pf) cudaEventDestroy(c->ev_pf);
    if (c->pf_buf) cudaFreeHost(c->pf_buf);
    for (auto& e : c->ev_chunk)
        if (e) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    for (auto& e : c->prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto& e : c->upd_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    delete c;
}

int coru_ctx_set_stream(coru_ctx* c, void* s) {
    if (!c) return fail(CORU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    return CORU_OK;
}

int coru_ctx_set_profiling(coru_ctx* c, int enable) {
    if (!c) return fail(CORU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    c->prof = enable != 0;
    c->prof_used = 0;
    c->prof_flops = c->prof_bytes = 0;
    return CORU_OK;
}

int coru_ctx_last_f64_engine(coru_ctx* c) { return c ? c->last_f64_engine : -1; }
int64_t coru_ctx_graph_replays(coru_ctx* c) { return c ? c->graph_replays : -1; }

int coru_ctx_profile_apass_exclusive(coru_ctx* c, double* total_ms, int64_t* launches) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    double ms = 0;
    int64_t n = 0;
    for (size_t i = 0; i < c->prof_used; ++i) {
        if (i < c->prof_shared.size() && c->prof_shared[i]) continue;
        float t = 0;
        CORU_CUDA(cudaEventSynchronize(c->prof_events[i].second));
        CORU_CUDA(cudaEventElapsedTime(&t, c->prof_events[i].first, c->prof_events[i].second));
        ms += t;
        ++n;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = n;
    return CORU_OK;
}

int coru_ctx_profile_apass(coru_ctx* c, double* total_ms, int64_t* launches, double* flops, double* bytes) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    double ms = 0;
    for (size_t i = 0; i < c->prof_used; ++i) {
        float t = 0;
        CORU_CUDA(cudaEventSynchronize(c->prof_events[i].second));
        CORU_CUDA(cudaEventElapsedTime(&t, c->prof_events[i].first, c->prof_events[i].second));
        ms += t;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = int64_t(c->prof_used);
    if (flops) *flops = c->prof_flops;
    if (bytes) *bytes = c->prof_bytes;
    c->prof_used = 0;
    c->prof_flops = c->prof_bytes = 0;
    return CORU_OK;
}

int coru_ctx_profile_rpca_update(coru_ctx* c, double* total_ms, int64_t* launches, double* flops, double* bytes) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    double ms = 0;
    for (size_t i = 0; i < c->upd_used; ++i) {
        float t = 0;
        CORU_CUDA(cudaEventSynchronize(c->upd_events[i].second));
        CORU_CUDA(cudaEventElapsedTime(&t, c->upd_events[i].first, c->upd_events[i].second));
        ms += t;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = int64_t(c->upd_used);
    if (flops) *flops = c->upd_flops;
    if (bytes) *bytes = c->upd_bytes;
    c->upd_used = 0;
    c->upd_flops = c->upd_bytes = 0;
    return CORU_OK;
}

int coru_ctx_set_host_threads(coru_ctx* c, int threads) {
    if (!c || threads < 1) return fail(CORU_EINVAL, "bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    c->host_threads = threads;
    return CORU_OK;
}

int coru_ctx_set_phi_mode(coru_ctx* c, int mode) {
    if (!c || (mode != CORU_PHI_DEVICE && mode != CORU_PHI_HOST_EXACT)) return fail(CORU_EINVAL, "bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    c->phi_mode = mode;
    return CORU_OK;
}

int coru_ctx_set_f32_path(coru_ctx* c, int mode) {
    if (!c || mode < CORU_F32_AUTO || mode > CORU_F32_TC) return fail(CORU_EINVAL, "bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    c->f32_path = mode;
    return CORU_OK;
}

int coru_ctx_set_f64_engine(coru_ctx* c, int mode) {
    if (!c || mode < CORU_F64_AUTO || mode > CORU_F64_OZAKI_HYBRID) return fail(CORU_EINVAL, "bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    c->f64_engine = mode;
    return CORU_OK;
}

int coru_ctx_set_wide_qr(coru_ctx* c, int enable) {
    if (!c) return fail(CORU_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    c->wide_qr = enable != 0;
    return CORU_OK;
}

int coru_comm_unique_id(unsigned char id[128]) {
    Nccl* api = nccl();
    if (!api) return fail(CORU_ENCCL, "NCCL unavailable");
    ncclUniqueId u;
    CORU_NCCL(api->GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return CORU_OK;
}

int coru_ctx_init_comm(coru_ctx* c, int rank, int world, const unsigned char id[128]) {
    CORU_TRY(enter(c));
    if (world < 1 || rank < 0 || rank >= world) return fail(CORU_EINVAL, "bad rank/world");
    std::lock_guard<std::mutex> lk(c->mu);
    // world 1 needs no communicator; CORU_NCCL_WORLD1 (tests) builds one anyway so the NCCL plumbing
    // (dlopen, init, all-reduce on the library's stream) runs on a single-GPU box
    if (world == 1 && !getenv("CORU_NCCL_WORLD1")) {
        c->rank = 0;
        c->world = 1;
        return CORU_OK;
    }
    Nccl* api = nccl();
    if (!api) return fail(CORU_ENCCL, "NCCL unavailable");
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    CORU_NCCL(api->CommInitRank(&c->comm, world, u, rank));
    c->rank = rank;
    c->world = world;
    return CORU_OK;
}

coru_threadcomm* coru_threadcomm_create(int world) {
    if (world < 1) return nullptr;
    return new coru_threadcomm(world);
}

void coru_threadcomm_destroy(coru_threadcomm* g) { delete g; }

int coru_ctx_init_threadcomm(coru_ctx* c, coru_threadcomm* g, int rank) {
    CORU_TRY(enter(c));
    if (!g || rank < 0 || rank >= g->world) return fail(CORU_EINVAL, "bad thread group / rank");
    // The group's collectives read the other ranks' device buffers directly (k_sum_slots, the
    // all-gather copies): every pair of devices in the group must reach each other. Same device:
    // nothing to do; different devices: enable peer access both ways or refuse (CORU_ENOTSUP).
    {
        std::lock_guard<std::mutex> gl(g->mu);
        g->devices[size_t(rank)] = c->device;
        for (int r = 0; r < g->world; ++r) {
            const int other = g->devices[size_t(r)];
            if (other < 0 || other == c->device) continue;
            int a = 0, b = 0;
            cudaDeviceCanAccessPeer(&a, c->device, other);
            cudaDeviceCanAccessPeer(&b, other, c->device);
            if (!a || !b) {
                g->devices[size_t(rank)] = -1;
                return fail(CORU_ENOTSUP, "thread group spans devices without peer access (" +
                                              std::to_string(c->device) + " <-> " + std::to_string(other) + ")");
            }
            for (auto [from, to] : {std::pair<int, int>{c->device, other}, {other, c->device}}) {
                cudaSetDevice(from);
                const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                    cudaGetLastError();
                    cudaSetDevice(c->device);
                    g->devices[size_t(rank)] = -1;
                    return fail(CORU_ENOTSUP, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
                }
                cudaGetLastError();
            }
            cudaSetDevice(c->device);
        }
    }
    std::lock_guard<std::mutex> lk(c->mu);
    c->tcomm = g;
    c->rank = rank;
    c->world = g->world;
    return CORU_OK;
}

void coru_shard_rows(int64_t m, int rank, int world, int64_t* row0, int64_t* rows) {
    // Contiguous, balanced row blocks: rank g owns [g*m/G, (g+1)*m/G).
    const int64_t a = m * rank / world, b = m * (rank + 1) / world;
    if (row0) *row0 = a;
    if (rows) *rows = b - a;
}

int coru_corutv_f64_dev(coru_ctx* c, const double* A, int64_t m_local, int64_t m, int64_t n, int64_t lda,
                        int64_t ell, int q, int variant, uint64_t seed, uint64_t stream, coru_utv* out) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    return corutv_dev<double>(c, A, m_local, m, n, lda, ell, q, variant, seed, stream, out);
}

int coru_corutv_f32_dev(coru_ctx* c, const float* A, int64_t m_local, int64_t m, int64_t n, int64_t lda,
                        int64_t ell, int q, int variant, uint64_t seed, uint64_t stream, coru_utv* out) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    return corutv_dev<float>(c, A, m_local, m, n, lda, ell, q, variant, seed, stream, out);
}

int coru_corutv_f64(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t ell, int q, int variant,
                    uint64_t seed, uint64_t stream, double* U, double* T, double* V, int64_t* perm, int* lower,
                    int* warn) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    return corutv_host<double>(c, A, m, n, ell, q, variant, seed, stream, U, T, V, perm, lower, warn);
}

int coru_corutv_f64_ooc(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q,
                        int variant, uint64_t seed, uint64_t stream, int64_t chunk_rows, coru_utv* out) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    return corutv_ooc<double>(c, A, m, n, lda, ell, q, variant, seed, stream, chunk_rows, out);
}

// CORU binary matrix (io.hpp:67-95): "CORU", rows, cols (u64 little-endian), rows·cols fp64 LE row-major.
int coru_read_matrix_bin_header(const char* path, int64_t* rows, int64_t* cols) {
    if (!path || !rows || !cols) return fail(CORU_EINVAL, "null argument");
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return fail(CORU_EIO, std::string("cannot open ") + path);
    struct stat stt {};
    unsigned char h[20];
    const bool ok = fstat(fd, &stt) == 0 && pread(fd, h, 20, 0) == 20;
    close(fd);
    auto u64 = [&](int o) {
        uint64_t v = 0;
        for (int b = 7; b >= 0; --b) v = (v << 8) | h[o + b];
        return v;
    };
    if (!ok || stt.st_size < 20 || std::memcmp(h, "CORU", 4) != 0)
        return fail(CORU_EIO, std::string(path) + ": not a CORU binary matrix");
    const uint64_t r = u64(4), cc = u64(12);
    if (r == 0 || cc == 0 || cc > (uint64_t(1) << 40) / r || uint64_t(stt.st_size) != 20 + 8 * r * cc)
        return fail(CORU_EIO, std::string(path) + ": truncated or malformed CORU file");
    *rows = int64_t(r);
    *cols = int64_t(cc);
    return CORU_OK;
}

int coru_corutv_f64_file(coru_ctx* c, const char* path, int64_t ell, int q, int variant, uint64_t seed,
                         uint64_t stream, int64_t chunk_rows, coru_utv* out) {
    CORU_TRY(enter(c));
    int64_t m = 0, n = 0;
    CORU_TRY(coru_read_matrix_bin_header(path, &m, &n));
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return fail(CORU_EIO, std::string("cannot open ") + path);
    const size_t len = 20 + size_t(m) * size_t(n) * 8;
    void* base = mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
    close(fd);
    if (base == MAP_FAILED) return fail(CORU_EIO, std::string("mmap failed: ") + path);
    madvise(base, len, MADV_SEQUENTIAL);
    // the payload starts at byte 20 (4 mod 8): it is only ever copied as bytes (cudaMemcpy2DAsync)
    const double* A = reinterpret_cast<const double*>(static_cast<const char*>(base) + 20);
    int rc;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        rc = corutv_ooc<double>(c, A, m, n, n, ell, q, variant, seed, stream, chunk_rows, out);
    }
    munmap(base, len);
    if (rc == CORU_EINVAL && std::string(coru_last_error()) == "Matrix: non-finite entry")
        return fail(CORU_EIO, std::string(path) + ": Matrix: non-finite entry");
    return rc;
}

int coru_corutv_f32_ooc(coru_ctx* c, const float* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q,
                        int variant, uint64_t seed, uint64_t stream, int64_t chunk_rows, coru_utv* out) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    return corutv_ooc<float>(c, A, m, n, lda, ell, q, variant, seed, stream, chunk_rows, out);
}

int coru_corutv_f32(coru_ctx* c, const float* A, int64_t m, int64_t n, int64_t ell, int q, int variant,
                    uint64_t seed, uint64_t stream, float* U, float* T, float* V, int64_t* perm, int* lower,
                    int* warn) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    return corutv_host<float>(c, A, m, n, ell, q, variant, seed, stream, U, T, V, perm, lower, warn);
}

int coru_sketch_bases_f64_dev(coru_ctx* c, const double* A, int64_t m_local, int64_t m, int64_t n, int64_t lda,
                              int64_t ell, int q, uint64_t seed, uint64_t stream, double* Q1, int64_t ldq1,
                              double* Q2, int64_t ldq2, double* C1, int64_t ldc1, double* C2prev, int64_t ldc2,
                              int* warn) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_params(m, n, ell, q));
    if (!A || !Q1 || !Q2) return fail(CORU_EINVAL, "null argument");
    if (c->world <= 1 && m_local != m) return fail(CORU_EINVAL, "m_local != m without a communicator");
    Request<double> r;
    r.A = A;
    r.lda = lda;
    r.rows = m_local;
    r.cols = n;
    r.d = int(ell);
    r.q = q;
    r.seed = seed;
    r.stream = stream;
    r.mode = Mode::Sketch;
    r.q1 = Q1;
    r.ldq1 = ldq1;
    r.q2 = Q2;
    r.ldq2 = ldq2;
    r.c1 = C1;
    r.ldc1 = ldc1;
    r.c2p = C2prev;
    r.ldc2 = ldc2;
    r.warn_host = warn;
    return run<double>(c, r);
}

int coru_sketch_bases_f64(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t ell, int q, uint64_t seed,
                          uint64_t stream, double* Q1, double* Q2, double* C1, double* C2prev, int* warn) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_params(m, n, ell, q));
    if (!A || !Q1 || !Q2) return fail(CORU_EINVAL, "null argument");
    Carver head{nullptr, 0};
    double *a_d = head.take<double>(m * n), *q1_d = head.take<double>(m * ell), *q2_d = head.take<double>(n * ell),
           *c1_d = head.take<double>(m * ell), *c2_d = head.take<double>(n * ell);
    const size_t head_bytes = (head.off + 255) / 256 * 256;
    Request<double> r;
    r.rows = m;
    r.cols = n;
    r.d = int(ell);
    r.q = q;
    r.seed = seed;
    r.stream = stream;
    r.mode = Mode::Sketch;
    r.c2p = reinterpret_cast<double*>(1);  // request the c2_prev buffer in the layout
    {
        Work<double> w;
        Carver meas{nullptr, head_bytes};
        w.layout(meas, c, r, int(round_up(ell, 8)));
        CORU_TRY(ensure_arena(c, meas.off));
    }
    Carver cv{c->arena, 0};
    a_d = cv.take<double>(m * n);
    q1_d = cv.take<double>(m * ell);
    q2_d = cv.take<double>(n * ell);
    c1_d = cv.take<double>(m * ell);
    c2_d = cv.take<double>(n * ell);
    cudaStream_t st = c->stream;
    CORU_CUDA(cudaMemcpyAsync(a_d, A, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
    r.A = a_d;
    r.lda = n;
    r.q1 = q1_d;
    r.ldq1 = ell;
    r.q2 = q2_d;
    r.ldq2 = ell;
    r.c1 = c1_d;
    r.ldc1 = ell;
    r.c2p = c2_d;
    r.ldc2 = ell;
    r.warn_host = warn;
    CORU_TRY(run<double>(c, r, head_bytes));
    CORU_CUDA(cudaMemcpyAsync(Q1, q1_d, sizeof(double) * m * ell, cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaMemcpyAsync(Q2, q2_d, sizeof(double) * n * ell, cudaMemcpyDeviceToHost, st));
    if (C1) CORU_CUDA(cudaMemcpyAsync(C1, c1_d, sizeof(double) * m * ell, cudaMemcpyDeviceToHost, st));
    if (C2prev) CORU_CUDA(cudaMemcpyAsync(C2prev, c2_d, sizeof(double) * n * ell, cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    return CORU_OK;
}

int coru_project_f64_dev(coru_ctx* c, const double* A, int64_t m_local, int64_t n, int64_t lda, const double* Q1,
                         int64_t ldq1, const double* Q2, int64_t ldq2, int64_t ell, double* D, int64_t ldd) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (ell < 1 || !A || !Q1 || !Q2 || !D) return fail(CORU_EINVAL, "bad argument");
    const int d = int(ell);
    Carver meas{nullptr, 0};
    auto lay = [&](Carver& cv, double*& W, double*& Mb, double*& ws, int64_t& wse) {
        W = cv.take<double>(m_local * ell);
        Mb = cv.take<double>(ell * ell);
        wse = std::max(gemm_ws<double>(Op::N, m_local, n, d, c->num_sms), gemm_ws<double>(Op::T, d, m_local, d, c->num_sms));
        ws = cv.take<double>(wse);
    };
    double *W, *Mb, *ws;
    int64_t wse;
    lay(meas, W, Mb, ws, wse);
    CORU_TRY(ensure_arena(c, meas.off));
    Carver cv{c->arena, 0};
    lay(cv, W, Mb, ws, wse);
    CORU_TRY(gemm<double>(c, Op::N, A, lda, Q2, ldq2, W, d, m_local, n, d, ws, wse));
    CORU_TRY(gemm<double>(c, Op::T, Q1, ldq1, W, d, Mb, d, d, m_local, d, ws, wse));
    CORU_TRY(allreduce<double>(c, Mb, size_t(d) * d));
    CORU_CUDA(copy_block<double>(Mb, d, D, ldd, d, d, c->stream));
    ++g_launches;
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

int coru_gaussian(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out, int threads) {
    if (rows < 1 || cols < 1 || !out) return fail(CORU_EINVAL, "Matrix: dimensions must be positive");
    gaussian_host<double>(rows, cols, seed, stream, out, cols, threads, 0);
    return CORU_OK;
}

int coru_gaussian_f64_dev(coru_ctx* c, int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out,
                          int64_t ldo) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (rows < 1 || cols < 1 || ldo < cols || !out) return fail(CORU_EINVAL, "Matrix: dimensions must be positive");
    uint64_t s4[4];
    seed_state_words(seed, stream, s4);
    CORU_CUDA(gaussian_dev<double>(rows, cols, s4, out, ldo, c->stream));
    ++g_launches;
    return CORU_OK;
}

int coru_gemm_f64_dev(coru_ctx* c, int op, const double* A, int64_t lda, const double* X, int64_t ldx, double* C,
                      int64_t ldc, int64_t rows, int64_t K, int64_t N) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (rows < 1 || K < 1 || N < 1 || N > 4096 || (op != 0 && op != 1)) return fail(CORU_EINVAL, "bad gemm shape");
    if (ldx % 2 != 0 || reinterpret_cast<uintptr_t>(X) % 16 != 0)
        return fail(CORU_EINVAL, "X must be 16-byte aligned with an even leading dimension");
    const Op o = op ? Op::T : Op::N;
    const int64_t wse = gemm_ws<double>(o, rows, K, int(N), c->num_sms);
    CORU_TRY(ensure_arena(c, size_t(wse) * 8 + 256));
    // A is an A-pass operand here: the Ozaki engine takes it when the shape qualifies
    const int64_t srows = o == Op::N ? rows : K, scols = o == Op::N ? K : rows;
    CORU_TRY(oz_prepare(c, A, lda, srows, scols, 1, int(N)));
    const int rc = gemm<double>(c, o, A, lda, X, ldx, C, ldc, rows, K, int(N), reinterpret_cast<double*>(c->arena), wse);
    c->oz_a = nullptr;
    CORU_TRY(rc);
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

int coru_gemm_f32_dev(coru_ctx* c, int op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C,
                      int64_t ldc, int64_t rows, int64_t K, int64_t N) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (rows < 1 || K < 1 || N < 1 || (op != 0 && op != 1)) return fail(CORU_EINVAL, "bad gemm shape");
    const Op o = op ? Op::T : Op::N;
    const int64_t wse = gemm_ws<float>(o, rows, K, int(N), c->num_sms);
    CORU_TRY(ensure_arena(c, size_t(wse) * 4 + 256));
    CORU_TRY(gemm<float>(c, o, A, lda, X, ldx, C, ldc, rows, K, int(N), reinterpret_cast<float*>(c->arena), wse));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

int coru_pinv_f64_dev(coru_ctx* c, const double* Y, int64_t ldy, int64_t n, double* P, int64_t ldp, int* converged) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (n < 1 || ldy < n || ldp < n) return fail(CORU_EINVAL, "pinv: bad shape");
    CORU_TRY(ensure_arena(c, size_t(pinv_ws_doubles(int(n))) * sizeof(double) + 256));
    double* ws = reinterpret_cast<double*>(c->arena);
    int* conv_d = reinterpret_cast<int*>(ws + pinv_ws_doubles(int(n)));
    CORU_CUDA(pinv_square<double>(Y, ldy, int(n), P, ldp, ws, conv_d, c->max_smem, c->stream));
    g_launches += kPinvLaunches;
    int conv = 0;
    CORU_CUDA(cudaMemcpyAsync(&conv, conv_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    if (converged) *converged = conv;
    return CORU_OK;
}


/* ---- SVD-based baselines (baselines.hpp:43-71) ---------------------------------------------- */
int coru_svd_f64_dev(coru_ctx* c, const double* Y, int64_t ldy, int64_t n, double* U, int64_t ldu, double* S,
                     double* V, int64_t ldv, int* converged) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (n < 1 || ldy < n || ldu < n || ldv < n || !Y || !U || !S || !V) return fail(CORU_EINVAL, "svd: bad shape");
    CORU_TRY(ensure_arena(c, size_t(pinv_ws_doubles(int(n))) * sizeof(double) + 256));
    double* ws = reinterpret_cast<double*>(c->arena);
    int* conv_d = reinterpret_cast<int*>(ws + pinv_ws_doubles(int(n)));
    CORU_CUDA(svd_square<double>(Y, ldy, int(n), U, ldu, S, V, ldv, ws, conv_d, c->max_smem, c->stream));
    g_launches += kSvdLaunches;
    int conv = 0;
    CORU_CUDA(cudaMemcpyAsync(&conv, conv_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    if (converged) *converged = conv;
    return CORU_OK;
}

int coru_tsr_svd_f64_dev(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t ell, uint64_t seed,
                         uint64_t stream, double* U, int64_t ldu, double* S, double* V, int64_t ldv, int* converged) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_tsr(m, n, ell));
    if (!A || !U || !S || !V || lda < n) return fail(CORU_EINVAL, "bad argument");
    if (c->world > 1) return fail(CORU_EINVAL, "tsr_svd: single-GPU entry");
    size_t need = 0;
    CORU_TRY(tsr_impl(c, A, m, n, lda, int(ell), seed, stream, U, ldu, S, V, ldv, converged, 0, &need));
    CORU_TRY(ensure_arena(c, need));
    return tsr_impl(c, A, m, n, lda, int(ell), seed, stream, U, ldu, S, V, ldv, converged, 0);
}

int coru_tsr_svd_f64(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t ell, uint64_t seed, uint64_t stream,
                     double* U, double* S, double* V, int* converged) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_tsr(m, n, ell));
    if (!A || !U || !S || !V) return fail(CORU_EINVAL, "null argument");
    if (c->world > 1) return fail(CORU_EINVAL, "host-buffer entry is single-GPU");
    Carver head{nullptr, 0};
    double *a_d, *u_d, *s_d, *v_d;
    int* f_d;
    auto lay = [&](Carver& cv) {
        a_d = cv.take<double>(m * n);
        u_d = cv.take<double>(m * ell);
        s_d = cv.take<double>(ell);
        v_d = cv.take<double>(n * ell);
        f_d = cv.take<int>(4);
    };
    lay(head);
    const size_t hb = (head.off + 255) / 256 * 256;
    size_t need = 0;
    CORU_TRY(tsr_impl(c, nullptr, m, n, n, int(ell), seed, stream, nullptr, ell, nullptr, nullptr, ell, nullptr, hb,
                      &need));
    CORU_TRY(ensure_arena(c, need));
    Carver cv{c->arena, 0};
    lay(cv);
    CORU_TRY(upload_checked(c, A, m * n, a_d, f_d));
    CORU_TRY(tsr_impl(c, a_d, m, n, n, int(ell), seed, stream, u_d, ell, s_d, v_d, ell, converged, hb));
    cudaStream_t st = c->stream;
    CORU_CUDA(cudaMemcpyAsync(U, u_d, sizeof(double) * m * ell, cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaMemcpyAsync(S, s_d, sizeof(double) * ell, cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaMemcpyAsync(V, v_d, sizeof(double) * n * ell, cudaMemcpyDeviceToHost, st));
    CORU_CUDA(cudaStreamSynchronize(st));
    return CORU_OK;
}

int coru_sor_svd_f64_dev(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t k, int64_t ell,
                         int q, uint64_t seed, uint64_t stream, double* L, int64_t ldl) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_sor(m, n, k, ell, q));
    if (!A || !L || lda < n || ldl < n) return fail(CORU_EINVAL, "bad argument");
    if (c->world > 1) return fail(CORU_EINVAL, "sor_svd: single-GPU entry");
    size_t need = 0;
    CORU_TRY(sor_impl(c, A, m, n, lda, int(k), int(ell), q, seed, stream, L, ldl, 0, &need));
    CORU_TRY(ensure_arena(c, need));
    return sor_impl(c, A, m, n, lda, int(k), int(ell), q, seed, stream, L, ldl, 0);
}

int coru_sor_svd_f64(coru_ctx* c, const double* A, int64_t m, int64_t n, int64_t k, int64_t ell, int q, uint64_t seed,
                     uint64_t stream, double* L) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_sor(m, n, k, ell, q));
    if (!A || !L) return fail(CORU_EINVAL, "null argument");
    if (c->world > 1) return fail(CORU_EINVAL, "host-buffer entry is single-GPU");
    Carver head{nullptr, 0};
    double *a_d, *l_d;
    int* f_d;
    auto lay = [&](Carver& cv) {
        a_d = cv.take<double>(m * n);
        l_d = cv.take<double>(m * n);
        f_d = cv.take<int>(4);
    };
    lay(head);
    const size_t hb = (head.off + 255) / 256 * 256;
    size_t need = 0;
    CORU_TRY(sor_impl(c, nullptr, m, n, n, int(k), int(ell), q, seed, stream, nullptr, n, hb, &need));
    CORU_TRY(ensure_arena(c, need));
    Carver cv{c->arena, 0};
    lay(cv);
    CORU_TRY(upload_checked(c, A, m * n, a_d, f_d));
    CORU_TRY(sor_impl(c, a_d, m, n, n, int(k), int(ell), q, seed, stream, l_d, n, hb));
    CORU_CUDA(cudaMemcpyAsync(L, l_d, sizeof(double) * m * n, cudaMemcpyDeviceToHost, c->stream));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

int coru_tsqr_f64_dev(coru_ctx* c, const double* B, int64_t ldb, int64_t m, int64_t n, double* Q, int64_t ldq,
                      double* R, int64_t ldr) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (n < 1 || m <= n) return fail(CORU_EINVAL, "householder_qr: requires rows > cols for TSQR");
    TsqrBufs<double> tb;
    Carver meas{nullptr, 0};
    tb.carve(meas, m, int(n), c->max_smem, c->num_sms, c->wide_qr);
    double* r = meas.take<double>(n * n);
    CORU_TRY(ensure_arena(c, meas.off));
    Carver cv{c->arena, 0};
    tb.carve(cv, m, int(n), c->max_smem, c->num_sms, c->wide_qr);
    r = cv.take<double>(n * n);
    CORU_TRY(tb.factor(B, ldb, r, c->stream));
    CORU_TRY(tb.form_q(nullptr, Q, ldq, c->stream));
    CORU_CUDA(copy_block<double>(r, n, R, ldr, n, int(n), c->stream));
    ++g_launches;
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

int coru_qrcp_f64_dev(coru_ctx* c, const double* M, int64_t ldm, int64_t n, double* Q, int64_t ldq, double* R,
                      int64_t ldr, int64_t* perm) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    if (n < 1 || n > 544) return fail(CORU_EINVAL, "qrcp: 1 <= n <= 544");
    Carver meas{nullptr, 0};
    meas.take<double>(qrcp_scratch_elems(int(n)));
    meas.take<int64_t>(n);
    CORU_TRY(ensure_arena(c, meas.off));
    Carver cv{c->arena, 0};
    double* scr = cv.take<double>(qrcp_scratch_elems(int(n)));
    int64_t* p = cv.take<int64_t>(n);
    CORU_CUDA(qrcp<double>(M, int(ldm), int(n), Q, int(ldq), R, int(ldr), p, scr, c->max_smem, c->stream));
    ++g_launches;
    CORU_CUDA(cudaMemcpyAsync(perm, p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

void coru_rpca_config_default(coru_rpca_config* cf) {
    if (!cf) return;
    cf->lambda = 0.0;
    cf->mu0 = 0.0;
    cf->rho = 1.5;
    cf->mu_bar = 0.0;
    cf->tol = 1e-5;
    cf->max_iter = 50;
    cf->inner = CORU_RPCA_CORUTV;
    cf->corutv_ell = 0;
    cf->corutv_q = 1;
    cf->thresholding = CORU_COR_SOFT;
}

int coru_alm_rpca_f64_dev(coru_ctx* c, const double* M, int64_t m, int64_t n, int64_t ldm, const coru_rpca_config* cf,
                          uint64_t seed, uint64_t stream, double* L, int64_t ldl, double* S, int64_t lds,
                          coru_rpca_result* res) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_rpca(cf, m, n));
    if (!M || !L || !S || !res || ldm < n || ldl < n || lds < n) return fail(CORU_EINVAL, "bad argument");
    if (c->world > 1) return fail(CORU_EINVAL, "alm_rpca: single-GPU entry");
    size_t need = 0;
    CORU_TRY(rpca_impl(c, M, m, n, ldm, *cf, seed, stream, L, ldl, S, lds, res, 0, &need));
    CORU_TRY(ensure_arena(c, need));
    return rpca_impl(c, M, m, n, ldm, *cf, seed, stream, L, ldl, S, lds, res, 0);
}

int coru_alm_rpca_f64(coru_ctx* c, const double* M, int64_t m, int64_t n, const coru_rpca_config* cf, uint64_t seed,
                      uint64_t stream, double* L, double* S, coru_rpca_result* res) {
    CORU_TRY(enter(c));
    std::lock_guard<std::mutex> lk(c->mu);
    CORU_TRY(check_rpca(cf, m, n));
    if (!M || !L || !S || !res) return fail(CORU_EINVAL, "null argument");
    if (c->world > 1) return fail(CORU_EINVAL, "host-buffer entry is single-GPU");
    Carver head{nullptr, 0};
    double *m_d, *l_d, *s_d;
    int* f_d;
    auto lay = [&](Carver& cv) {
        m_d = cv.take<double>(m * n);
        l_d = cv.take<double>(m * n);
        s_d = cv.take<double>(m * n);
        f_d = cv.take<int>(4);
    };
    lay(head);
    const size_t hb = (head.off + 255) / 256 * 256;
    size_t need = 0;
    CORU_TRY(rpca_impl(c, nullptr, m, n, n, *cf, seed, stream, nullptr, n, nullptr, n, res, hb, &need));
    CORU_TRY(ensure_arena(c, need));
    Carver cv{c->arena, 0};
    lay(cv);
    CORU_TRY(upload_checked(c, M, m * n, m_d, f_d));
    CORU_TRY(rpca_impl(c, m_d, m, n, n, *cf, seed, stream, l_d, n, s_d, n, res, hb));
    CORU_CUDA(cudaMemcpyAsync(L, l_d, sizeof(double) * m * n, cudaMemcpyDeviceToHost, c->stream));
    CORU_CUDA(cudaMemcpyAsync(S, s_d, sizeof(double) * m * n, cudaMemcpyDeviceToHost, c->stream));
    CORU_CUDA(cudaStreamSynchronize(c->stream));
    return CORU_OK;
}

}  // extern "C"
