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
constexpr int kPinvLaunches = 2;

}  // namespace coru_gpu
