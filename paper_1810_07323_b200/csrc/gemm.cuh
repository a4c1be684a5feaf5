// Skinny A-pass GEMMs of CoR-UTV.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace coru_gpu {

// C[Mo x N] = op(A) · X where
//   op = N : op(A) = A   (A is Mo x K, row-major, lda)          — B1 = A·B2, W = A·Q2, U = Q1·Q_M
//   op = T : op(A) = A^T (A is K x Mo, row-major, lda; no copy) — B2 = A^T·B1, M = Q1^T·W
// X is K x N row-major (ldx), C is Mo x N row-major (ldc). N is the (padded) sketch width.
// Deterministic: split-K partials are reduced in a fixed order; no floating-point atomics.
enum class Op { N = 0, T = 1 };

struct GemmPlan {
    int bm = 0, bn = 0, splits = 1;  // fp64: splits = stream-K CTA count
    int max_seg = 1;                 // fp64 stream-K: max CTAs sharing one tile
    bool fixup = false;              // fp64 stream-K: some tile is split across CTAs
    int cfg = -1;                    // fp64: kernel configuration id (gemm_f64.cu table)
    int num_sms = 148;
    int64_t ws_elems = 0;            // workspace (partials) needed, in elements
    int groups = 1;                  // fp64: grouped stream-K, one CTA group per n-tile (splits per group)
};

GemmPlan plan_gemm_f64(Op op, int64_t Mo, int64_t K, int N, int num_sms);
// Explicit configuration (cfg < 0: default); for tuning tools.
GemmPlan plan_gemm_f64_cfg(Op op, int64_t Mo, int64_t K, int N, int num_sms, int cfg);
int gemm_f64_num_configs();
// Tooling: cap the stream-K CTAs per output tile (0 = planner default); affects every later plan.
void gemm_f64_set_split_cap(int cap);
// `ws` must hold plan.ws_elems doubles when plan.splits > 1.
cudaError_t gemm_f64(Op op, const double* A, int64_t lda, const double* X, int64_t ldx, double* C,
                     int64_t ldc, int64_t Mo, int64_t K, int N, const GemmPlan& plan, double* ws,
                     cudaStream_t stream);

GemmPlan plan_gemm_f32(Op op, int64_t Mo, int64_t K, int N, int num_sms);
cudaError_t gemm_f32(Op op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C, int64_t ldc,
                     int64_t Mo, int64_t K, int N, const GemmPlan& plan, float* ws, cudaStream_t stream);

// fp32 A-pass on tcgen05 tensor cores (3xTF32, TMA + TMEM; gemm_tc32.cu). `ws` must hold
// gemm_tc32_ws_elems floats. Call only when gemm_tc32_supported().
bool gemm_tc32_supported(Op op, const float* A, int64_t lda, int64_t Mo, int64_t K, int N);
bool gemm_tc32_eligible(int64_t Mo, int64_t K, int N);
int64_t gemm_tc32_ws_elems(int64_t Mo, int64_t K, int N, int num_sms);
int gemm_tc32_launches(int64_t Mo, int64_t K, int N, int num_sms);
cudaError_t gemm_tc32(Op op, const float* A, int64_t lda, const float* X, int64_t ldx, float* C, int64_t ldc,
                      int64_t Mo, int64_t K, int N, float* ws, int num_sms, int max_smem, cudaStream_t st);

// fp64 A-pass on the INT8 tensor cores (tcgen05 kind::i8, Ozaki-scheme emulation; gemm_oz.cu).
// eA: per output row of op(A), the exponent E with max |row| < 2^E (gemm_oz_exponents: erow for
// op N, ecol for op T). `ws` must hold gemm_oz_ws_bytes bytes.
bool gemm_oz_eligible(int64_t Mo, int64_t K, int N);
bool gemm_oz_supported(Op op, const double* A, int64_t lda, int64_t Mo, int64_t K, int N);
size_t gemm_oz_ws_bytes(int64_t Mo, int64_t K, int N, int num_sms);
cudaError_t gemm_oz_exponents(const double* A, int64_t lda, int64_t rows, int64_t cols, int* erow, int* ecol,
                              cudaStream_t st);
// The same pass in pieces, for a matrix that arrives in row chunks (the host entry's upload
// pipeline): begin (clear) -> rows [r0, r0 + nrows) as they become resident -> end (finish).
cudaError_t gemm_oz_exponents_begin(int64_t rows, int64_t cols, int* erow, int* ecol, cudaStream_t st);
cudaError_t gemm_oz_exponents_rows(const double* A, int64_t lda, int64_t r0, int64_t nrows, int64_t cols, int* erow,
                                   int* ecol, cudaStream_t st);
cudaError_t gemm_oz_exponents_end(int64_t rows, int64_t cols, int* erow, int* ecol, cudaStream_t st);
// Digit planes of a prepared matrix (gemm_oz_planes): the 7 slices of every entry, converted once
// per decomposition — PN (row scales, K-major for op N) followed by PT (column scales, transposed:
// K-major for op T) in one buffer of pn_bytes + pt_bytes.
struct OzPlaneDims {
    int64_t ldn = 0, ldt = 0;       // bytes per plane row
    size_t pn_bytes = 0, pt_bytes = 0;
};
OzPlaneDims gemm_oz_plane_dims(int64_t rows, int64_t cols);
cudaError_t gemm_oz_planes(const double* A, int64_t lda, int64_t rows, int64_t cols, const int* erow, const int* ecol,
                           uint8_t* planes, cudaStream_t st);
struct OzPlanes {
    const uint8_t* p = nullptr;     // plane set matching the op: [7][rows][ld]
    int64_t ld = 0, rows = 0;       // rows = rows of the plane set (output rows of op(A) for the whole matrix)
};
// pl != nullptr: A-pass over the planes (A, lda unused); else A is converted inside the kernel.
// store != nullptr (op N, in-kernel conversion only): the pass also writes the row-scaled digit
// planes of the rows it covers to `store`, for later op-N passes to run with pl = store.
cudaError_t gemm_oz(Op op, const double* A, int64_t lda, const OzPlanes* pl, const int* eA, const double* X,
                    int64_t ldx, double* C, int64_t ldc, int64_t Mo, int64_t K, int N, void* ws, int num_sms,
                    cudaStream_t st, const OzPlanes* store = nullptr);
int gemm_oz_launches(int64_t Mo, int64_t K, int N, int num_sms);

}  // namespace coru_gpu
