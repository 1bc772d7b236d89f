// gace_kernels.h -- launchers of the sm_100a kernels (internal, not the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include "gace_plan.h"

namespace gace {

constexpr int kMaxSmem = 227 * 1024;   // opt-in dynamic shared memory per CTA on sm_100a

cudaError_t launch_probe(const ProbeParams &P, bool sample, bool i64, int grid, cudaStream_t s);
cudaError_t launch_finalize(const FinParams &F, cudaStream_t s);
cudaError_t launch_minmax(const void *col, int dtype, uint64_t n, long long *mm, int sms, cudaStream_t s);
cudaError_t launch_hll_ceilings(long long dl, unsigned long long span, bool is64, uint32_t *scratch32,
                                uint8_t *out8, int sms, cudaStream_t s);
cudaError_t launch_sample_mask(uint64_t nrows, uint64_t row0, uint64_t seed, uint64_t thr, bool all,
                               unsigned long long *bits, cudaStream_t s);

}  // namespace gace
