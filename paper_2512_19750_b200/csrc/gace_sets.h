// gace_sets.h -- device-side layout of the candidate-set probe (internal, not the C-ABI).
//
// What it computes: PAPER.md §IV-H "Experiment D: Replacing Dynamic Sampling (Key-Only +
// Bitmask)" (lines 250-270): M candidate predicate sets of K predicates each; per set, the
// number of (sampled) rows on which every member predicate holds (SPEC.md evaluate_bitmasks:
// "per-set count = popcount of AND-ed bitmaps"; shared predicates evaluated once).
//
// B200 design (DESIGN.md §6 "Candidate sets"): the planner turns each probed column's member
// predicates into sorted breakpoints (buckets on which every predicate is constant) and, per
// bucket, a set-satisfaction mask sat_c[b] = {m : every member of set m on column c holds on
// bucket b} (sets with no member on c: all ones).  A row satisfies set m iff bit m survives
// the AND over columns of sat_c[bucket_c(row)] -- C lookups per row whatever K and M are.
// The per-row masks are counted with bit-sliced per-lane counters and a warp bit-matrix
// transpose + popcount every 28 rows (no per-row atomics).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gace {

constexpr int kSetsMaxCols = 8;       // probed columns per call (GACE_MAX_PROBED_COLS)
constexpr int kSetsMaxWords = 8;      // 32-set words: nsets <= 256
constexpr int kSetsThreads = 1024;     // one CTA per SM (<= 64 registers)
constexpr uint32_t kSetsCellB0Bits = 20;          // cell word: b0 | n << 20 (| kSetsImpure)
constexpr uint32_t kSetsCellNMax = (1u << 11) - 1;
constexpr uint32_t kSetsImpure = 0x80000000u;     // folded plans: cell holds breakpoints

struct SetsCol {
    const void *ptr;        // column values of this launch (16-byte aligned)
    int64_t dlo;            // value domain minimum (attach-time): offsets u = v - dlo
    uint32_t is64;          // 1: int64 column
    uint32_t shift;         // cell = u >> shift
    uint32_t cell_off;      // u32 index of the cell table in shared memory
    uint32_t bps_off;       // u64 index of the breakpoint offsets (sorted, u = t - dlo)
    uint32_t sat_off;       // u32 index of sat[bucket][W]
    uint32_t pad;
};

struct SetsParams {
    SetsCol col[kSetsMaxCols];
    uint32_t ncols;
    uint32_t W;             // 32-set words
    uint32_t image_u4;      // shared-memory image size (uint4)
    uint32_t fold;          // W == 1, nsets <= 31: breakpoint-free cells hold their sat mask
    const uint4 *image;     // cells | breakpoints | sat masks
    uint64_t nrows;         // rows of this launch
    uint64_t row0;          // global id of the first row (sample bit)
    uint64_t seed;
    uint64_t thr;           // keep iff u(seed, r) < thr  (ignored when !SAMPLE)
    unsigned long long *g_counts;   // [W * 32] u64
    unsigned long long *g_nsamp;
};

cudaError_t launch_sets(const SetsParams &P, bool sample, bool i64, int grid, cudaStream_t s);

}  // namespace gace
