// Rank-revealing QR of the d x d core and the lift.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace coru_gpu {

// Column-pivoted QR M·P = Q_M·T of a d x d row-major M (ldm). Outputs: Q_M (d x d, ldq),
// T (d x d upper with exact zeros below, ldt), perm[d] (int64). `scratch` must hold
// qrcp_scratch_elems(d) elements when d is too wide for shared memory.
template <typename T>
cudaError_t qrcp(const T* M, int ldm, int d, T* Q, int ldq, T* Tout, int ldt, int64_t* perm, T* scratch,
                 int max_smem, cudaStream_t st);
int64_t qrcp_scratch_elems(int d);

// V(:, j) = Q2(:, perm[j])  (corutv.hpp:95-97); V is n x d (ldv), Q2 n x d (ldq).
template <typename T>
cudaError_t gather_columns(const T* Q2, int64_t ldq, const int64_t* perm, int64_t n, int d, T* V, int64_t ldv,
                           cudaStream_t st);

// flag = |R(d-1,d-1)| <= 1e-14·|R(0,0)|   (corutv.hpp:61-64)
template <typename T>
cudaError_t conditioning_flag(const T* R, int ldr, int d, int* flag, cudaStream_t st);

// Copy a rows x cols block between row-major matrices (device).
template <typename T>
cudaError_t copy_block(const T* src, int64_t lds, T* dst, int64_t ldd, int64_t rows, int cols, cudaStream_t st);

// flag = 1 if any of the n entries is non-finite (the Matrix constructor check, matrix.hpp:29-31).
template <typename T>
cudaError_t any_nonfinite(const T* A, int64_t n, int* flag, cudaStream_t st);
// Same check, accumulating into a flag the caller zeroed (chunked uploads).
template <typename T>
cudaError_t any_nonfinite_acc(const T* A, int64_t n, int* flag, cudaStream_t st);

// Transpose a d x d row-major block: dst(i,j) = src(j,i)  (ULV orientation, corutv.hpp:84-86).
template <typename T>
cudaError_t transpose_square(const T* src, int lds, T* dst, int ldd, int d, cudaStream_t st);

}  // namespace coru_gpu
