// Tall-skinny QR (TSQR) of the sketches B1 (m x d) and B2 (n x d) — SURVEY.md §2.2 K3.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace coru_gpu {

// One level of the R-reduction tree: `rows` input rows split into `nb` contiguous blocks
// (block b = rows [rows*b/nb, rows*(b+1)/nb), each with more than d rows).
struct TsqrLevel {
    int64_t rows = 0;
    int nb = 0;
    int rbmax = 0;     // max rows in a block
    int ldv = 0;       // column stride of a block's stored reflectors (>= rbmax)
    int64_t v_off = 0;     // offset (elements) of this level's reflector store in the V arena
    int64_t beta_off = 0;  // offset of the betas
    int64_t r_off = 0;     // offset of the stacked R (nb*d x d, ld = d) output in the R arena
    int64_t t_off = 0;     // offset of the per-block compact-WY T factors (blocked path)
    enum Kind { kBlockedSmem = 0, kBlockedGlobal = 1, kWide = 2, kReg = 3 };
    Kind kind = kBlockedSmem;  // which kernel pair factors / forms Q for this level
    bool blocked = false;  // panel-blocked compact-WY kernels (else the unblocked column pipeline)
    bool smem = true;      // working block lives in shared memory (else in the V arena, L2)
};

struct TsqrPlan {
    int64_t m = 0;
    int d = 0;
    std::vector<TsqrLevel> levels;
    bool blocked = false;  // level 0 uses the blocked kernels
    int64_t v_elems = 0, beta_elems = 0, r_elems = 0, t_elems = 0;
    int max_smem = 0;
    size_t elem_bytes = 8;
};

TsqrPlan plan_tsqr(int64_t m, int d, size_t elem_bytes, int max_smem_bytes, int num_sms = 148);

// Factor B (m x d, row-major, ldb) through the tree. R (d x d, row-major, upper, exact zeros
// below) is written to r_out (ld = d) — on device.
template <typename T>
// gate (device int, may be null): when it reads 0 the kernels return at once (CholeskyQR2 already
// produced this QR, cholqr.cu).
cudaError_t tsqr_factor(const TsqrPlan& p, const T* B, int64_t ldb, T* v_arena, T* beta_arena, T* t_arena,
                        T* r_arena, T* r_out, cudaStream_t st, const int* gate = nullptr);

// Form the explicit Q (m x d, row-major, ldq) from a factored tree. If q_top is non-null it is the
// d x d (row-major, ld = d) block that multiplies the tree's top-level Q from the right — used for
// the cross-rank top level (Q_g = Q_local_tree · Q_global[g*d:(g+1)*d, :]); null means identity.
template <typename T>
cudaError_t tsqr_form_q(const TsqrPlan& p, const T* q_top, T* v_arena, T* beta_arena, T* t_arena, T* scratch, T* Q,
                        int64_t ldq, int max_smem, cudaStream_t st, const int* gate = nullptr);

// scratch of tsqr_form_q: working blocks (wide path), T-product buffers and two level buffers.
int64_t tsqr_scratch_elems(const TsqrPlan& p);

}  // namespace coru_gpu
