// gace_plan.h -- internal plan layout shared by the host planner (gace_host.cpp)
// and the sm_100a kernels (gace_kernels.cu).  Not part of the C-ABI.
//
// The planner turns a predicate batch into, per probed column ("slot"):
//   * the sorted breakpoints T of all its predicates (interval ends lo and hi+1,
//     clipped to the column's value domain), so that every predicate is a
//     contiguous bucket range of  bucket(v) = #{t in T : t <= v};
//   * a two-level lookup table over the offset u = v - base that resolves
//     bucket(v) with one shared-memory load and one compare;
//   * a u32 shared-memory histogram over the buckets (counts are prefix sums);
// and, per pair of probed columns carrying cross-column pairs ("group"), a 2-D
// histogram over the sub-buckets of only the pair-relevant predicates (joints are
// rectangle sums).  HLL registers live in shared memory as u8[4096] per column.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>   // uint2 / uint4
#include <stdint.h>
#else                       // NVRTC (gace_jit.cpp): built-in vector types, no libc headers
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#endif

namespace gace {

constexpr int kMaxSlots = 8;           // GACE_MAX_PROBED_COLS
constexpr int kMaxGroups = 28;         // unordered slot pairs
constexpr int kHllP = 12;
constexpr int kHllM = 1 << kHllP;
constexpr int kThreads = 512;          // probe CTA size (one CTA per SM, <= 128 registers)
constexpr uint32_t kNoThr = 0xFFFFFFFFu;
constexpr uint32_t kSpecial = 0x80000000u;  // entry is a level-2 pointer or a list
constexpr uint32_t kList = 0x40000000u;     // special entry is a short sorted list
constexpr uint32_t kBaseMask = 0x00FFFFFFu;
constexpr uint32_t kListMax = 63;
constexpr uint32_t kNone = 0xFFFFFFFFu;

#if defined(__CUDACC__)
#define GACE_HD __host__ __device__ __forceinline__
#else
#define GACE_HD inline
#endif

// Byte address (in shared memory) of the bucket counter of offset u.  `M` reads the
// table image: M.u4(i) / M.u32(i) (shared memory in the kernel; a bounds-checked copy
// in gace_debug_buckets).  Entry formats: see SlotParams below.
template <class Mem>
GACE_HD uint32_t lut_lookup(const Mem &M, uint32_t lut_idx, uint32_t s1, uint32_t u) {
    uint32_t s = s1;
    uint4 e = M.u4(lut_idx + (u >> s));
    while ((e.x & (kSpecial | kList)) == kSpecial) {        // block of sub-cells (nested)
        const uint32_t sc = (e.x >> 24) & 63u;
        e = M.u4(e.y + ((u & ((1u << s) - 1u)) >> sc));
        s = sc;
    }
    if (e.x & kList) {
        uint32_t b = e.x & kBaseMask;
        const uint32_t n = (e.x >> 24) & 63u;
        for (uint32_t i = 0; i < n; ++i) b += (u >= M.u32(e.y + i)) ? 4u : 0u;
        return b;
    }
    return e.x + (u > e.y ? 4u : 0u) + (u > e.z ? 4u : 0u) + (u > e.w ? 4u : 0u);
}

enum SlotMode : uint8_t { MODE_LUT = 0, MODE_SEARCH = 1, MODE_NOPRED = 2 };

// LUT entry (16 bytes), over the offset u = v - base of one column.  Buckets are named
// by the shared-memory BYTE address of their u32 counter (no scaling on the hot path).
//   direct : x = address of the cell's first bucket, y <= z <= w = up to three
//            thresholds (unused: ~0); bucket = x + 4 * #{t in (y, z, w) : u > t}
//   nested : x = kSpecial | sc << 24, y = uint4 index of a block of sub-cells of size
//            2^sc; sub-entry = T[y + ((u mod cell size) >> sc)] (any of the three kinds)
//   list   : x = kSpecial | kList | n << 24 | first bucket address, y = u32 index of n
//            sorted breakpoint offsets t, bucket = first + 4 * #{t : u >= t}
struct SlotParams {
    const void *ptr;        // device column base for this launch
    const int64_t *bps;     // MODE_SEARCH: sorted breakpoints (device)
    int64_t base;           // u = (uint32)(v - base)
    int64_t clamp_lo;       // CLAMP kernels: v = min(max(v, clamp_lo), clamp_hi)
    int64_t clamp_hi;
    uint32_t nbp;           // MODE_SEARCH: number of breakpoints
    uint32_t s1;            // level-1 cell = u >> s1
    uint32_t cell_mask;     // (1 << s1) - 1
    uint32_t lut_idx;       // level-1 table: uint4 index into shared memory
    uint32_t l2_idx;        // nested sub-cell blocks: uint4 index into shared memory
    uint32_t hist_addr;     // byte address of bucket 0 of this column's histogram
    uint32_t hll_idx;       // u32 index of this column's u32[4096] HLL registers, or kNone
    uint8_t dtype;          // 0 = int32, 1 = int64
    uint8_t mode;           // SlotMode
    uint8_t has_hll;
    uint8_t pad;
};

struct GroupParams {
    int32_t mapA_adj;       // byte address of mapA minus hist_addr of slot a: map entry of a
    int32_t mapB_adj;       //   bucket at [bucket address + adj]; values are grid byte offsets
    uint16_t dbeg, dend;    // this column pair's per-row ("direct") pairs: direct[dbeg .. dend)
    uint8_t a, b;           // slots, a < b
    uint8_t has_grid;       // 2-D grid in shared memory (else all its pairs are direct)
    uint8_t pad;
};

// Cross-column pair evaluated per row (fallback when a group's 2-D grid does not fit).
struct DirectPair {
    uint32_t la, ha;        // bucket-address interval of the predicate on slot a (la > ha: empty)
    uint32_t lb, hb;        // ... on slot b
    uint32_t nega, negb;
    uint32_t acc_idx;       // u32 index of its counter in shared memory
};

struct ProbeParams {
    SlotParams slot[kMaxSlots];
    GroupParams grp[kMaxGroups];
    uint32_t nslots;
    uint32_t ngroups;                      // column pairs carrying cross-column pairs
    uint32_t ndirect;
    const DirectPair *direct;              // device
    const uint4 *image;                    // device: tables copied into shared memory
    uint32_t image_u4;                     // image size in 16-byte units
    uint32_t acc_idx;                      // u32 index where the zeroed accumulators start
    uint32_t acc_words;                    // number of u32 accumulators
    uint32_t hll_off;                      // byte offset of the u32 HLL register block (nh * 4096 u32)
    uint32_t hll_bytes;                    // nh * 4096: bytes of the packed u8 registers output
    uint32_t smem_bytes;                   // total dynamic shared memory
    unsigned long long *g_acc;             // u64[acc_words], summed over CTAs (and launches)
    uint8_t *g_hll_part;                   // [part_slot][hll_bytes] per-CTA register partials
    unsigned long long *g_nsamp;
    uint64_t nrows;                        // rows in this launch
    uint64_t row0;                         // global id of the launch's first row
    uint64_t thr;                          // floor(rate * 2^64)
    uint64_t seed;
    uint32_t sample_all;                   // rate == 1
    uint32_t part_merge;                   // 1: max-merge into existing per-CTA partials (later chunk launches)
    uint32_t clamp;                        // clamp keys into each slot's [clamp_lo, clamp_hi]
    uint32_t dbg;                          // ablation bits (env GACE_ABLATE; 0 in production):
                                           // 1 no HLL raise, 2 no histogram adds, 4 no grid adds, 8 no HLL
};

// ---------------------------------------------------------------- finalize

enum FinJobKind : uint32_t { JOB_HIST = 0, JOB_SAT = 1 };

struct FinJob {
    uint32_t kind;
    uint32_t src;           // index into g_acc
    uint32_t dst;           // index into g_pre
    uint32_t na, nb;        // HIST: nb buckets (na unused); SAT: na x nb grid
};

enum FinPairKind : uint32_t { PAIR_SAME = 0, PAIR_GRID = 1, PAIR_DIRECT = 2 };

struct FinPred {
    uint32_t pre;           // g_pre index of the column's exclusive prefix (nb + 1 values)
    uint32_t lo, hi;        // bucket interval (lo > hi: empty)
    uint32_t neg;
};

struct FinPair {
    uint32_t kind;
    uint32_t pre;           // SAME: 1-D prefix; GRID: SAT (row stride nb + 1); DIRECT: g_acc index
    uint32_t na, nb;        // GRID: grid extent
    uint32_t li, hi, lj, hj;// SAME: bucket intervals; GRID: i on the A side, j on the B side
    uint32_t negi, negj;
};

struct FinParams {
    const FinJob *jobs;
    uint32_t njobs;
    uint32_t hll_bytes;
    uint32_t nparts;        // number of per-CTA HLL partials
    uint32_t hll_blocks;
    const unsigned long long *g_acc;
    unsigned long long *g_pre;
    const uint8_t *g_hll_part;
    const unsigned long long *g_nsamp;
    const FinPred *preds;
    uint32_t npreds;
    const FinPair *pairs;
    uint32_t npairs;
    unsigned long long *out;    // [1 + npreds + npairs]: n_sampled, counts, joints
    uint8_t *out_regs;          // [hll_bytes]
};

}  // namespace gace
