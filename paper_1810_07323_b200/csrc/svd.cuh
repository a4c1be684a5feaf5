// Pseudo-inverse of the d x d sketch core for DVariant::approx (corutv.hpp:91-92):
// pinv (svd.hpp:167-187) via one-sided Jacobi SVD (svd.hpp:31-134), in fp64 for both dtypes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace coru_gpu {

// P (d x d, ldp) = pinv(Y) for a square d x d row-major Y (ldy). Singular values at or below
// d·eps·sigma_1 are dropped (pinv's default tolerance, svd.hpp:184-187). `ws` holds
// pinv_ws_doubles(d) doubles. Two launches: the Jacobi sweeps (one CTA) and the assembly
// P = (V·Σ⁺)·Uᵀ (tiled over the grid). *converged (device, optional) receives the number of sweeps
// used (0 when the 60-sweep cap was hit).
template <typename T>
cudaError_t pinv_square(const T* Y, int64_t ldy, int d, T* P, int64_t ldp, double* ws, int* converged, int max_smem,
                        cudaStream_t st);
int64_t pinv_ws_doubles(int d);

// svd (svd.hpp:141-161) of a square d x d row-major Y: U, V (d x d row-major), sigma[d] non-increasing,
// zero-sigma u columns completed from the canonical basis (svd.hpp:98-121). Same workspace as
// pinv_square; afterwards `ws` still holds the sorted factors for svd_truncate_core.
template <typename T>
cudaError_t svd_square(const T* Y, int64_t ldy, int d, T* U, int64_t ldu, T* sigma, T* V, int64_t ldv, double* ws,
                       int* converged, int max_smem, cudaStream_t st);
// C (d x d, ldc) = u(:, 1:k)·diag(sigma_1..k)·v(:, 1:k)^T from the factors svd_square left in `ws`
// (svd_truncate, baselines.hpp:14-20).
template <typename T>
cudaError_t svd_truncate_core(const double* ws, int d, int k, T* C, int64_t ldc, cudaStream_t st);
// svt's core (rpca.hpp:30-40): C = u(:, 1:R)·diag(sigma_r - delta)·v(:, 1:R)^T with R = #{leading
// sigma_r > delta}, from the factors svd_square left in `ws`; R is written to *rank_out (device).
template <typename T>
cudaError_t svt_core(const double* ws, int d, double delta, T* C, int64_t ldc, int* rank_out, cudaStream_t st);
// The factors of svd (svd.hpp:141-161) left in `ws` only (sorted sigma, ut rows = u columns, vs rows =
// v columns), computed like the preconditioned pinv: Y·P = Q·R, one-sided Jacobi of R^T, factors
// permuted / rotated back — about half the sweeps of the plain square Jacobi on graded matrices; the
// same factors to rounding. Falls back to the plain Jacobi for d < 8 or d > 544. 4 launches.
template <typename T>
cudaError_t svd_factors_precond(const T* Y, int64_t ldy, int d, double* ws, int max_smem, cudaStream_t st);
constexpr int kSvdLaunches = 2;
constexpr int kPinvLaunches = 5;  // widen, QRCP, Jacobi, fix, assemble

}  // namespace coru_gpu
