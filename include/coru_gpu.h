/*
 * coru_gpu — C-ABI of the B200-native CoR-UTV hot path.
 *
 * Drop-in boundary for the reference's decomposition entry point and its sketch stage:
 *
 *   coru::corutv(const Matrix& a, size_t ell, int q, DVariant variant, RngSeed seed)
 *       -> UtvApprox{u, t, v, ell, q, variant, seed, lower, conditioning_warning}
 *       /root/reference/proj/include/coru/corutv.hpp:79-100 (UtvApprox :23-34)
 *   coru::detail::sketch_bases(const Matrix& a, size_t ell, int q, RngSeed seed)
 *       -> SketchBases{q1, q2, c1, c2_prev, conditioning_warning}
 *       /root/reference/proj/include/coru/corutv.hpp:42-65
 *   the projection D = (q1^T a) q2                      corutv.hpp:90
 *   coru::gaussian(rows, cols, seed)                    rng.hpp:107-112
 *
 * The reference is a header-only C++ library with no FFI; a C++ caller uses the header-only
 * wrapper include/coru_gpu.hpp (same names and types as the reference), other languages bind
 * these symbols directly. Plain pointers and sizes only.
 *
 * Matrices are dense row-major (the layout of coru::Matrix, matrix.hpp:44-45) with an explicit
 * leading dimension. "_dev" entry points take device pointers; the others take host pointers
 * and copy in and out inside the call. There is no CPU fallback: without a usable sm_100 GPU
 * every entry point fails with CORU_ECUDA.
 *
 * Errors mirror the reference: CORU_EINVAL is std::invalid_argument (corutv.hpp:68-70,81 — ell < 1,
 * ell >= min(rows, cols), q < 0; matrix.hpp:29-31 — non-finite host input), everything else maps
 * to std::runtime_error in the C++ wrapper. coru_last_error() returns the calling thread's message.
 */
#ifndef CORU_GPU_H
#define CORU_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CORU_GPU_ABI_VERSION 1

enum coru_status {
    CORU_OK = 0,
    CORU_EINVAL = 1,  /* std::invalid_argument in the reference */
    CORU_ECUDA = 2,   /* CUDA runtime / launch failure, or no sm_100 device */
    CORU_ENCCL = 3,   /* NCCL failure (multi-GPU) */
    CORU_ENOMEM = 4,  /* device or pinned-host allocation failed */
    CORU_ENOTSUP = 5, /* valid in the reference, not provided by this build */
    CORU_EIO = 6      /* coru::IoError (io.hpp): unreadable / malformed CORU file */
};

/* DVariant (corutv.hpp:17): exact = D from one more pass over A (corutv.hpp:90); approx = D from the
 * sketches, (Q1^T C1)·pinv(Q2^T C2prev) (corutv.hpp:91-92), with the pinv computed in fp64. */
enum coru_variant { CORU_D_EXACT = 0, CORU_D_APPROX = 1 };

/* Opaque per-device context: stream, workspace arena, pinned staging, optional communicator.
 * Calls on one context are serialised by an internal mutex; use one context per host thread
 * for concurrent decompositions (the reference is re-entrant; coru_cli.cpp:171). */
typedef struct coru_ctx coru_ctx;

int coru_abi_version(void);
const char* coru_last_error(void);

int coru_ctx_create(int device, coru_ctx** out);
void coru_ctx_destroy(coru_ctx* ctx);
/* Run on the caller's cudaStream_t (NULL restores the context-owned non-blocking stream; pass
 * cudaStreamLegacy for the legacy default stream). */
int coru_ctx_set_stream(coru_ctx* ctx, void* cuda_stream);
/* Host threads used for the bit-exact Gaussian test matrix (default: hardware concurrency). */
int coru_ctx_set_host_threads(coru_ctx* ctx, int threads);
/* Where corutv draws Φ (corutv.hpp:51):
 *   CORU_PHI_HOST_EXACT (default): generated on the host with the host libm, bit-identical to the
 *     reference's gaussian() (rng.hpp:86-112), by the worker pool in row chunks whose H2D copies
 *     overlap the generation of the next chunk;
 *   CORU_PHI_DEVICE (opt-in): generated on the GPU — the reference's xoshiro256++ word stream
 *     bit-for-bit, Box–Muller with the device log/sincos (entries within a few ulp of the host's). */
enum { CORU_PHI_DEVICE = 0, CORU_PHI_HOST_EXACT = 1 };
int coru_ctx_set_phi_mode(coru_ctx* ctx, int mode);
/* fp32 A-pass engine (the fp32 configuration; matmul at corutv.hpp:55,57,90):
 *   CORU_F32_AUTO (default): tcgen05 3xTF32 tensor-core kernel (TMA + TMEM) for A-pass-sized
 *     products, CUDA-core FFMA otherwise;  CORU_F32_SIMT / CORU_F32_TC: force one engine
 *     (CORU_F32_TC still uses FFMA where the tensor-core kernel cannot take the shape). */
enum { CORU_F32_AUTO = 0, CORU_F32_SIMT = 1, CORU_F32_TC = 2 };
/* fp64 A-pass engine (matmul at corutv.hpp:55,57,90 over the caller's A):
 *   CORU_F64_AUTO (default): INT8 tensor cores (tcgen05.mma kind::i8) with the Ozaki scheme —
 *     7 digit slices per operand against per-row / per-column power-of-two scales, exact int32
 *     slice products, fp64 recombination (~2^-55 relative error vs. row-max x column-max);
 *     FP64 DMMA for shapes it cannot take and for every non-A-pass product;
 *     A is either converted to digits inside every A-pass kernel (few passes, narrow sketch) or
 *     once per decomposition into its digit planes (14 bytes per entry of extra device memory)
 *     that every pass then streams — chosen from (passes over A) x (N-chunks of the sketch); in
 *     between (two or more A·X passes), hybrid: the first A·X pass converts in the kernel and
 *     also writes the row-scaled planes (7 bytes per entry), the later A·X passes stream them,
 *     the A^T·Y passes convert in the kernel. All variants produce the same bits;
 *   CORU_F64_DMMA: FP64 DMMA for everything;
 *   CORU_F64_OZAKI_INLINE / CORU_F64_OZAKI_PLANES / CORU_F64_OZAKI_HYBRID: the Ozaki engine with the
 *     conversion forced into the A-pass kernel / the once-per-decomposition digit planes / hybrid. */
enum {
    CORU_F64_AUTO = 0, CORU_F64_DMMA = 1, CORU_F64_OZAKI_INLINE = 2, CORU_F64_OZAKI_PLANES = 3,
    CORU_F64_OZAKI_HYBRID = 4
};
int coru_ctx_set_f64_engine(coru_ctx* ctx, int mode);
/* Engine the last fp64 decomposition's A-passes ran on: 0 = FP64 DMMA, 1 = Ozaki with in-kernel
 * digits, 2 = Ozaki over digit planes, 3 = Ozaki hybrid (bench evidence: which roofline applies). */
int coru_ctx_last_f64_engine(coru_ctx* ctx);
/* Small in-core single-GPU decompositions (rows·cols <= 2^24, ell <= 112, default engines, profiling
 * off, the context's own stream or any non-legacy stream set with coru_ctx_set_stream) are replayed
 * from a CUDA graph from the third call with the same device buffers and parameters on (the seed
 * may change: Φ is generated per call); CORU_NO_GRAPH=1 disables it.
 * Returns the number of replays so far (bench evidence). */
int64_t coru_ctx_graph_replays(coru_ctx* ctx);
int coru_ctx_set_f32_path(coru_ctx* ctx, int mode);
/* QR of wide sketches (more than 128 columns; householder_qr at corutv.hpp:59-60): 1 (default) =
 * CholeskyQR2 in fp64 with a device-side fall-back to the Householder tree when the sketch is
 * ill-conditioned (estimated cond > 1e6) or the Cholesky breaks down; 0 = Householder tree only. */
int coru_ctx_set_wide_qr(coru_ctx* ctx, int enable);

/* ---- multi-GPU: one process (and context) per GPU, A row-block sharded --------------------- */
/* Rank 0 creates the id and distributes it (e.g. torch.distributed broadcast); every rank then
 * calls coru_ctx_init_comm. NCCL is loaded at run time (libnccl.so.2). */
int coru_comm_unique_id(unsigned char id[128]);
int coru_ctx_init_comm(coru_ctx* ctx, int rank, int world, const unsigned char id[128]);
/* In-process alternative to NCCL: ranks are host threads of one process (one context each, on one
 * GPU or on peer-accessible GPUs); collectives are a stream sync + host barrier + fixed-order
 * device sum, deterministic and identical on every rank. coru_ctx_init_threadcomm enables peer
 * access between the new rank's device and every device already in the group, and returns
 * CORU_ENOTSUP if two of them cannot reach each other. */
typedef struct coru_threadcomm coru_threadcomm;
coru_threadcomm* coru_threadcomm_create(int world);
void coru_threadcomm_destroy(coru_threadcomm* group);
int coru_ctx_init_threadcomm(coru_ctx* ctx, coru_threadcomm* group, int rank);
/* Rows [*row0, *row0 + *rows) of an m-row matrix belong to `rank` of `world`. */
void coru_shard_rows(int64_t m, int rank, int world, int64_t* row0, int64_t* rows);

/* ---- the decomposition: corutv (corutv.hpp:79-100) ------------------------------------------ */
/* Output record (UtvApprox, corutv.hpp:23-34). u: rows(A) x ell (this rank's rows when sharded),
 * t: ell x ell (upper for URV, lower for ULV), v: cols(A) x ell. perm (optional, host) receives the
 * QRCP pivots of the core (V(:,j) = Q2(:,perm[j]), corutv.hpp:95-97). */
typedef struct {
    void* u;
    int64_t ldu;
    void* t;
    int64_t ldt;
    void* v;
    int64_t ldv;
    int64_t* perm;            /* host, ell entries, may be NULL */
    int lower;                /* out: 1 for the ULV orientation (rows(A) < cols(A)) */
    int conditioning_warning; /* out: |R1(ell,ell)| <= 1e-14 |R1(1,1)| (corutv.hpp:61-64) */
} coru_utv;

/* A: device, row-major, lda >= n. With a communicator, A is this rank's m_local rows of the
 * global m x n matrix (coru_shard_rows layout); without one, m_local == m. */
int coru_corutv_f64_dev(coru_ctx* ctx, const double* A, int64_t m_local, int64_t m, int64_t n, int64_t lda,
                        int64_t ell, int q, int variant, uint64_t seed, uint64_t stream, coru_utv* out);
int coru_corutv_f32_dev(coru_ctx* ctx, const float* A, int64_t m_local, int64_t m, int64_t n, int64_t lda,
                        int64_t ell, int q, int variant, uint64_t seed, uint64_t stream, coru_utv* out);

/* Host-buffer drop-in for coru::corutv: A host row-major m x n (dense); U (m x ell), T (ell x ell),
 * V (n x ell) host row-major dense; perm optional. Single GPU (the context's device). */
int coru_corutv_f64(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t ell, int q, int variant,
                    uint64_t seed, uint64_t stream, double* U, double* T, double* V, int64_t* perm, int* lower,
                    int* conditioning_warning);
int coru_corutv_f32(coru_ctx* ctx, const float* A, int64_t m, int64_t n, int64_t ell, int q, int variant,
                    uint64_t seed, uint64_t stream, float* U, float* T, float* V, int64_t* perm, int* lower,
                    int* conditioning_warning);

/* Out-of-core corutv (§8 f4; the paper's pass model for externally stored data):
 * A stays in HOST memory (row-major m x n, lda >= n) and is streamed to the GPU in row
 * chunks of chunk_rows rows (<= 0: ~512 MB per chunk) through a two-buffer device ring, the H2D of
 * chunk i+1 overlapping the GEMMs of chunk i. Each power round reads A once (c1 rows = A_i·c2 and
 * the partial A_i^T·c1_i from the same chunk, summed in chunk order), the exact-D projection once
 * more: q + 2 streams of A (exact) / q + 1 (approx) instead of 2q + 3 / 2q + 2 passes. Only the
 * sketches (m x ell, cols x ell) and two chunks live on the device, so A may exceed HBM. Pageable
 * host memory is page-locked for the duration of the call. Outputs as coru_corutv_*_dev (device
 * U, T, V; host pointers are also accepted: the call then copies the factors back). rows < cols
 * runs the ULV orientation (lower = 1, corutv.hpp:82-87) with two reads of A per power round (the
 * A^T-side partial sums must complete first). Deterministic; differs from the in-core path at
 * rounding level (chunk-ordered partial sums). */
int coru_corutv_f64_ooc(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q,
                        int variant, uint64_t seed, uint64_t stream, int64_t chunk_rows, coru_utv* out);
int coru_corutv_f32_ooc(coru_ctx* ctx, const float* A, int64_t m, int64_t n, int64_t lda, int64_t ell, int q,
                        int variant, uint64_t seed, uint64_t stream, int64_t chunk_rows, coru_utv* out);

/* CORU binary matrix files (write_matrix_bin / read_matrix_bin, io.hpp:67-95): "CORU", rows, cols as
 * u64 little-endian, then rows·cols fp64 little-endian row-major. The header reader validates the magic
 * and the exact file size (CORU_EIO with the reference's messages). The file entry memory-maps the
 * file and runs the out-of-core corutv on it directly (A never materialised in host RAM beyond the
 * page cache); non-finite entries return CORU_EIO like read_matrix_bin. U, T, V: device (or host)
 * buffers for rows x ell, ell x ell, cols x ell. */
int coru_read_matrix_bin_header(const char* path, int64_t* rows, int64_t* cols);
int coru_corutv_f64_file(coru_ctx* ctx, const char* path, int64_t ell, int q, int variant, uint64_t seed,
                         uint64_t stream, int64_t chunk_rows, coru_utv* out);

/* ---- the sketch stage: detail::sketch_bases (corutv.hpp:42-65) ------------------------------- */
/* Requires rows(A) >= cols(A) like the reference's callers (rpca.hpp:135, baselines.hpp:68).
 * Q1/C1: m_local x ell, Q2/C2prev: n x ell (device, row-major). C1 and C2prev may be NULL. */
int coru_sketch_bases_f64_dev(coru_ctx* ctx, const double* A, int64_t m_local, int64_t m, int64_t n, int64_t lda,
                              int64_t ell, int q, uint64_t seed, uint64_t stream, double* Q1, int64_t ldq1,
                              double* Q2, int64_t ldq2, double* C1, int64_t ldc1, double* C2prev, int64_t ldc2,
                              int* conditioning_warning);
int coru_sketch_bases_f64(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t ell, int q,
                          uint64_t seed, uint64_t stream, double* Q1, double* Q2, double* C1, double* C2prev,
                          int* conditioning_warning);

/* ---- the projection D = (Q1^T A) Q2 (corutv.hpp:90), summed over ranks ----------------------- */
int coru_project_f64_dev(coru_ctx* ctx, const double* A, int64_t m_local, int64_t n, int64_t lda, const double* Q1,
                         int64_t ldq1, const double* Q2, int64_t ldq2, int64_t ell, double* D, int64_t ldd);

/* ---- the test matrix Φ: gaussian(rows, cols, {seed, stream}) (rng.hpp:107-112), host --------- */
int coru_gaussian(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out, int threads);
/* Device variant (CORU_PHI_DEVICE's generator): out is a device pointer with leading dimension
 * ldo >= cols (padding columns are zeroed), enqueued on the context's stream. */
int coru_gaussian_f64_dev(coru_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, uint64_t stream, double* out,
                          int64_t ldo);

/* ---- kernel-level entry points (parity tests and benchmarks of the A-pass kernels) ----------- */
/* C (rows x N) = op(A) · X, op 0: A (rows x K), op 1: A^T with A (K x rows); device row-major. */
int coru_gemm_f64_dev(coru_ctx* ctx, int op, const double* A, int64_t lda, const double* X, int64_t ldx,
                      double* C, int64_t ldc, int64_t rows, int64_t K, int64_t N);
int coru_gemm_f32_dev(coru_ctx* ctx, int op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C,
                      int64_t ldc, int64_t rows, int64_t K, int64_t N);
/* householder_qr (qr.hpp:85-99) via TSQR: B (m x n, m > n) -> Q (m x n), R (n x n). Device. */
int coru_tsqr_f64_dev(coru_ctx* ctx, const double* B, int64_t ldb, int64_t m, int64_t n, double* Q, int64_t ldq,
                      double* R, int64_t ldr);
/* qrcp (qr.hpp:106-143) of a square n x n matrix: Q, R (n x n), perm (host, n). Device. */
int coru_qrcp_f64_dev(coru_ctx* ctx, const double* M, int64_t ldm, int64_t n, double* Q, int64_t ldq, double* R,
                      int64_t ldr, int64_t* perm);

/* pinv (svd.hpp:167-187) of a square n x n matrix via the one-sided Jacobi SVD (svd.hpp:31-134), the
 * core of DVariant::approx (corutv.hpp:91-92). Device Y, P (row-major); *converged (host, may be
 * NULL) = the number of Jacobi sweeps used, 0 when the 60-sweep cap was hit. */
int coru_pinv_f64_dev(coru_ctx* ctx, const double* Y, int64_t ldy, int64_t n, double* P, int64_t ldp, int* converged);

/* ---- SVD-based baselines that share the CoR-UTV kernels (baselines.hpp:43-71), fp64 ----------- */
/* svd (svd.hpp:141-161) of a square n x n matrix: U, V (n x n), S[n] non-increasing (device);
 * *converged (host, may be NULL) = Jacobi sweeps used, 0 when the 60-sweep cap was hit. */
int coru_svd_f64_dev(coru_ctx* ctx, const double* Y, int64_t ldy, int64_t n, double* U, int64_t ldu, double* S,
                     double* V, int64_t ldv, int* converged);
/* tsr_svd(a, ell, seed) (baselines.hpp:43-56): U m x ell, S[ell], V n x ell; Φ1, Φ2 from the
 * sub-streams (stream, stream + 1). EINVAL "tsr_svd: ell out of range" unless 1 <= ell < min(m, n). */
int coru_tsr_svd_f64_dev(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, int64_t ell, uint64_t seed,
                         uint64_t stream, double* U, int64_t ldu, double* S, double* V, int64_t ldv, int* converged);
int coru_tsr_svd_f64(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t ell, uint64_t seed, uint64_t stream,
                     double* U, double* S, double* V, int* converged);
/* sor_svd(a, k, ell, q, seed) (baselines.hpp:61-71): L (m x n) = Q1·trunc_k(svd(Q1^T A Q2))·Q2^T with
 * corutv's sketch (same seed -> same Q1, Q2). EINVAL as the reference: ell (corutv's checks),
 * 1 <= k <= ell, q >= 0. */
int coru_sor_svd_f64_dev(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, int64_t k, int64_t ell,
                         int q, uint64_t seed, uint64_t stream, double* L, int64_t ldl);
int coru_sor_svd_f64(coru_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t k, int64_t ell, int q, uint64_t seed,
                     uint64_t stream, double* L);

/* ---- robust PCA by ALM with the CoR-UTV inner step: alm_rpca (rpca.hpp:95-169), fp64 ---------- */
/* RpcaInner (rpca.hpp:53): only the CoR-UTV inner is provided; svt_exact (the full SVD of every
 * m x n iterate, rpca.hpp:117-120) returns CORU_ENOTSUP. */
enum coru_rpca_inner { CORU_RPCA_SVT_EXACT = 0, CORU_RPCA_CORUTV = 1 };
/* CorutvThresholding (rpca.hpp:58): soft = svt of the compressed core (rpca.hpp:135-139), hard =
 * cor_threshold (corutv.hpp:124-134, rpca.hpp:130-133). */
enum coru_rpca_threshold { CORU_COR_SOFT = 0, CORU_COR_HARD = 1 };
/* RpcaConfig (rpca.hpp:60-78), same fields, defaults and validation (CORU_EINVAL with the reference's
 * messages). Defaults that need an SVD of M or of the iterate — mu0 <= 0 (1.25/||M||_2) and
 * corutv_ell == 0 (predict_rank(X) + 2, per iteration) — are computed on the GPU from the Gram matrix
 * X^T X and need cols(M) <= 1024 (CORU_ENOTSUP beyond). */
typedef struct {
    double lambda;   /* <= 0: 1/sqrt(max(m, n)) */
    double mu0;      /* <= 0: 1.25/||M||_2 */
    double rho;      /* continuation factor, > 1 (reference default 1.5) */
    double mu_bar;   /* <= 0: mu0·1e7 */
    double tol;      /* > 0 (reference default 1e-5) */
    int max_iter;    /* >= 1 (reference default 50) */
    int inner;       /* coru_rpca_inner */
    int64_t corutv_ell; /* 0: predict_rank(X) + 2 each iteration */
    int corutv_q;       /* >= 0 (reference default 1) */
    int thresholding;   /* coru_rpca_threshold */
} coru_rpca_config;
/* Fills the reference's defaults (RpcaConfig{} with inner = corutv). */
void coru_rpca_config_default(coru_rpca_config* cfg);
/* RpcaResult (rpca.hpp:80-88) minus l and s (the caller's buffers). residuals: host, max_iter entries
 * (may be NULL); zeta_j = ||M - L_j - S_j||_F / ||M||_F. */
typedef struct {
    int iterations;
    double* residuals;
    int64_t rank_l;
    int64_t s_l0;
    int converged;
    int ell_clamped;
} coru_rpca_result;
/* M, L, S: device row-major m x n (ldm, ldl, lds >= n); M is never written. Iteration j draws its
 * sketch from substream({seed, stream}, j) (rpca.hpp:129). Single GPU. */
int coru_alm_rpca_f64_dev(coru_ctx* ctx, const double* M, int64_t m, int64_t n, int64_t ldm,
                          const coru_rpca_config* cfg, uint64_t seed, uint64_t stream, double* L, int64_t ldl,
                          double* S, int64_t lds, coru_rpca_result* res);
/* Host-buffer drop-in for coru::alm_rpca: M, L, S host row-major dense m x n. */
int coru_alm_rpca_f64(coru_ctx* ctx, const double* M, int64_t m, int64_t n, const coru_rpca_config* cfg,
                      uint64_t seed, uint64_t stream, double* L, double* S, coru_rpca_result* res);

/* A-pass profiling: when enabled, CUDA events are recorded on the launching stream around every
 * GEMM that streams the caller's A (the sketch, power and projection passes). The read call
 * returns the summed device time, the number of A-passes, and their algorithmic flops
 * (2·rows·cols·ell) and A bytes (rows·cols·sizeof(T)), then resets the counters. */
int coru_ctx_set_profiling(coru_ctx* ctx, int enable);
int coru_ctx_profile_apass(coru_ctx* ctx, double* total_ms, int64_t* launches, double* flops, double* bytes);
/* The same counters restricted to the A-passes that had the GPU to themselves — not issued while
 * the call's second stream runs QR kernels (the Q1 tree under the last A^T pass of tall sketches and
 * under the projection pass). Does not reset; call before coru_ctx_profile_apass. */
int coru_ctx_profile_apass_exclusive(coru_ctx* ctx, double* total_ms, int64_t* launches);
/* The same for the fused lift + ALM update kernel of alm_rpca: algorithmic flops 2·m·n·ell (the lift
 * L = Tp·V^T) and bytes 40·m·n per launch (read M, Y; write S, Y, X). */
int coru_ctx_profile_rpca_update(coru_ctx* ctx, double* total_ms, int64_t* launches, double* flops, double* bytes);

/* Number of this library's kernels launched by the calling thread since the last reset
 * (bench evidence: "gpu_launches"). */
int64_t coru_launch_count(int reset);
/* Test tooling: cap the stream-K CTAs per output tile of the FP64 DMMA GEMM planner
 * (0 = the planner's own choice). Process-wide; affects every later plan. */
void coru_debug_gemm_split_cap(int cap);

#ifdef __cplusplus
}
#endif

#endif /* CORU_GPU_H */
