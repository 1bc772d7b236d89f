// gace_merge.h -- fused cross-GPU merge over an NCCL symmetric window (gace_merge.cu;
// internal, not the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace gace {

struct MergeState;

// True if the loaded libnccl exports the device-API host calls (NCCL >= 2.28).
bool merge_available();
// Collective over the communicator's ranks: a symmetric window of `bytes` per rank and a
// device communicator with one LSA barrier.  False (with *err, nothing allocated) when the
// device API is missing or not every rank is load/store reachable.
bool merge_create(void *nccl_comm, int nranks, size_t bytes, MergeState **out, std::string *err);
void merge_destroy(MergeState *m);
// This rank's window (device memory): the finalize writes its packed result here.
void *merge_buffer(MergeState *m, size_t *bytes);
// Sum the `nwords` u64 counters at offset 0 and max the `regs_bytes` register bytes at
// regs_off over every rank's window into `out` (same layout), between two LSA barriers.
cudaError_t merge_launch(MergeState *m, uint32_t nwords, uint32_t regs_off, uint32_t regs_bytes, void *out,
                         cudaStream_t s);

}  // namespace gace
