// ALM robust PCA with the CoR-UTV inner step (rpca.hpp:95-169, §8 f2): the kernels around the
// shared sketch / projection / SVD kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace coru_gpu {

// Per-iteration scalars of one ALM step (rpca.hpp:113-150), computed on the host exactly as the
// reference does (inv_mu = 1/mu, shrink threshold lambda·inv_mu, next inv_mu = 1/min(rho·mu, mu_bar)).
struct RpcaStep {
    double inv_mu;       // 1/mu_j
    double mu;           // mu_j (multiplier update y += mu·resid)
    double thresh;       // lambda·inv_mu (S-step)
    double inv_mu_next;  // 1/mu_{j+1} (the next iterate X = M - S + Y/mu_{j+1})
};

// The lift fused with the ALM update. L = Tp·Vb^T (Tp m x d, Vb n x d, row-major) is formed tile by
// tile in registers and never written; the epilogue applies, per entry and in the reference's
// operation order without contraction,
//   w = (M - L) + Y·inv_mu;  S = shrink(w, thresh);  r = (M - L) - S;  Y += mu·r;
//   X = (M - S) + Y·inv_mu_next
// writing S, Y, X, and one partial sum of r² per CTA (fixed tile order: deterministic).
// lift_only: write L = Tp·Vb^T and nothing else (the final L of the solve).
cudaError_t rpca_lift_update(const double* Tp, int64_t ldt, const double* Vb, int64_t ldv, int d, int64_t m,
                             int64_t n, const double* M, int64_t ldm, double* Y, int64_t ldy, double* X, int64_t ldx,
                             double* S, int64_t lds, double* L, int64_t ldl, const RpcaStep& p, bool lift_only,
                             double* parts, int nparts, cudaStream_t st);
// Number of CTAs (= partial sums) rpca_lift_update and sumsq use for an m x n matrix.
int rpca_parts(int64_t m, int64_t n, int sms);

// cor_threshold's truncation (corutv.hpp:124-134 + truncate_rank_k :106-110): r = #{j : |T_jj| > delta};
// Tr = T with rows >= r (upper, URV) or columns >= r (lower, ULV) zeroed; r -> *rank_out (device).
cudaError_t cor_truncate(const double* T, int64_t ldt, int d, double delta, int lower, double* Tr, int64_t ldtr,
                         int* rank_out, cudaStream_t st);

// Partial sums of squares of an m x n row-major matrix (nparts CTAs), then their fixed-order total.
cudaError_t sumsq_parts(const double* A, int64_t lda, int64_t m, int64_t n, double* parts, int nparts,
                        cudaStream_t st);
cudaError_t sum_parts(const double* parts, int nparts, double* out, cudaStream_t st);

// Norms from the eigenvalues of the Gram matrix (its singular values, non-increasing, length p):
// out[0] = sqrt(sigma_1) (spectral norm), out[1] = sum_i sqrt(max(sigma_i, 0)) (nuclear norm), i increasing.
cudaError_t gram_norms(const double* sig, int p, double* out, cudaStream_t st);

// l0_count (norms.hpp:21-25): number of nonzero entries; *out (device, unsigned long long).
cudaError_t count_nonzero(const double* A, int64_t lda, int64_t m, int64_t n, unsigned long long* out,
                          cudaStream_t st);

}  // namespace coru_gpu
