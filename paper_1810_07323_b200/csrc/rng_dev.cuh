// Device Φ generator (rng_dev.cu) and the host helpers it shares with rng_host.cpp.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace coru_gpu {

// xoshiro256++ state for {seed, stream} (rng.hpp:41-61 seeding), rng_host.cpp.
void seed_state_words(uint64_t seed, uint64_t stream, uint64_t out[4]);

// rows x cols Gaussians, row-major element e -> out[(e / cols) * ldo + e % cols], padding columns
// [cols, ldo) zeroed. Same word stream as gaussian_host; values within a few ulp of it.
template <typename OutT>
cudaError_t gaussian_dev(int64_t rows, int64_t cols, const uint64_t state[4], OutT* out, int64_t ldo, cudaStream_t st);

}  // namespace coru_gpu
