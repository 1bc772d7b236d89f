// gace_jit.h -- NVRTC specialisation of the probe kernel (internal).
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "gace_plan.h"

namespace gace {

constexpr int kMaxSmemJit = 227 * 1024;

// True if NVRTC and the driver API could be loaded (else *why says which).
bool jit_available(std::string *why);

// Launch the probe kernel specialised for `shape_src` (a generated `struct JitShape`),
// compiling and caching it on first use for (device, shape).  Adds the compile time to
// *compile_ms.  Returns false (with *err) if compilation or launch failed; nothing has
// been launched in that case.
bool jit_launch(const ProbeParams &P, int device, const std::string &shape_src, int grid, cudaStream_t s,
                double *compile_ms, std::string *err);

// The specialised kernel for (device, shape), compiled and cached on first use; and a launch
// of a kernel obtained that way (tables keep the handle of their cached plan, so repeated
// probes skip regenerating the shape source and the cache lookup).
bool jit_get(int device, const std::string &shape_src, void **fn, double *compile_ms, std::string *err);
bool jit_launch_fn(void *fn, const ProbeParams &P, int grid, int threads, cudaStream_t s, std::string *err);

// Non-blocking: the cached kernel for (device, shape) if it is compiled.
bool jit_lookup(int device, const std::string &shape_src, void **fn);
// Queue a background compile of (device, shape) (no-op if cached or already queued); a later
// jit_lookup finds it once the worker thread has loaded it.
void jit_prefetch(int device, const std::string &shape_src);
// Wait until no background compile is queued or running (false on timeout).
bool jit_bg_wait(double timeout_ms);
void jit_bg_shutdown();     // stop the worker: queued compiles dropped, one in progress finished
void jit_bg_stats(uint64_t *done, uint64_t *failed, uint64_t *pending);

// NVRTC compile only (no device needed): the test hook gace_debug_jit_compile.
bool jit_compile_check(const std::string &shape_src, size_t *cubin_bytes, std::string *err);

size_t jit_cache_size();

}  // namespace gace
