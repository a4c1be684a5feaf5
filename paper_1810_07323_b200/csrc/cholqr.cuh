// Wide-sketch QR by CholeskyQR2 in fp64 with a device-side fall-back status (cholqr.cu).
#pragma once
#include <cstdint>
#include <functional>
#include <cuda_runtime.h>

namespace coru_gpu {

struct CholQrPlan {
    int64_t m = 0;
    int d = 0;
    int ldw = 0;                 // even row stride of the fp64 work matrices
    int64_t xd_elems = 0;        // fp64 copy of an fp32 sketch (0 for fp64)
    int64_t q1_elems = 0;        // first-pass Q (fp64)
    int64_t gram_ws = 0;         // gemm_f64 workspace (Gram and R2·R1)
    int64_t dd_elems = 0;        // one d x ldw fp64 matrix
    int64_t rinvd_elems = 0;     // inverses of the 32 x 32 diagonal blocks of R
};

// Wide sketches (d > 128) whose blocked Cholesky and row-block solve fit shared memory.
bool cholqr_applicable(int64_t m, int d, int max_smem);
CholQrPlan plan_cholqr(int64_t m, int d, size_t elem_bytes, int num_sms);
int64_t cholqr_ws_doubles(const CholQrPlan& p);

// R (d x d, row-major, ld d, exact zeros below) of B (m x d, ldb) by CholeskyQR2 in fp64.
// status (device int): 0 = CholeskyQR2 result valid; nonzero = ill-conditioned or breakdown —
// the caller's gated Householder kernels then overwrite R and Q.
// Row-sharded B (every rank holds m local rows of the same tall matrix): `reduce` sums a buffer of
// `count` doubles over the ranks in place on `st` (identical bytes on every rank); it is applied to
// the two Gram matrices, so R, the status and the triangular solves are those of the stacked matrix.
using CholQrReduce = std::function<cudaError_t(double* buf, size_t count)>;
template <typename T>
cudaError_t cholqr_factor(const CholQrPlan& p, const T* B, int64_t ldb, double* ws, int* status, T* r_out,
                          int max_smem, int num_sms, cudaStream_t st, const CholQrReduce* reduce = nullptr);
// Q = Q1 · R2^{-1} (m x d, ldq) from the state cholqr_factor left in ws.
template <typename T>
cudaError_t cholqr_form_q(const CholQrPlan& p, double* ws, T* Q, int64_t ldq, int num_sms, cudaStream_t st);
int cholqr_launches(int d);

}  // namespace coru_gpu
