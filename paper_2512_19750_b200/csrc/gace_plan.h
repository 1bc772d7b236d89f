// gace_plan.h -- internal plan layout shared by the host planner (gace_host.cpp), the
// sm_100a kernels (gace_kernels.cu, gace_probe.cuh) and NVRTC (gace_jit.cpp).  Not part
// of the C-ABI.
//
// The planner turns a predicate batch into, per probed column ("slot"):
//   * the sorted breakpoints T of all its predicates (interval ends lo and hi+1, clipped
//     to the column's value domain), so every predicate is a contiguous range of
//     bucket(v) = #{t in T : t <= v};
//   * a lookup table over the offset u = v - base that resolves bucket(v) with one
//     16-byte shared-memory load and three compares;
// and, per pair of probed columns carrying cross-column pairs ("group"), a 2-D histogram
// grid[bucket of the A column][sub-bucket of the B column], the sub-buckets being cut only
// by the B-side predicates of that group's pairs.  Joints are rectangle sums of the grid;
// the grid's row sums are the A column's bucket histogram, so a column that is the A side
// of a group needs no histogram of its own.  The sub-bucket of a column's primary B role
// is packed into its lookup-table entries.  HLL registers live in shared memory as u32.
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
#ifndef GACE_THREADS
#define GACE_THREADS 1024
#endif
// probe CTA size (one CTA per SM): 1024 threads of <= 64 registers; a specialised kernel of a
// plan whose row unit holds many key registers is compiled with 768 (<= 80 registers: the
// column-streamed keys of 8 columns spilled at 64; gace_host.cpp jit_threads)
constexpr int kThreads = GACE_THREADS;
// static shared memory of the probe kernels (skip-bound slices and limits, the sparse-sample
// row queues: gace_probe.cuh); the plan's dynamic shared memory gets the rest of the 227 KB.
// A full scan's kernels carry no row queue (1.5-2.5 KB static), so a plan with sample rate 1
// gets 9 KB more for its tables (finer level-1 cells, fewer boundary records)
constexpr int kStaticSmem = 12 * 1024;
constexpr int kStaticSmemFull = 3 * 1024;
#ifndef __CUDACC_RTC__     // host side only (NVRTC takes no unannotated functions)
constexpr int static_smem_reserve(bool sample) { return sample ? kStaticSmem : kStaticSmemFull; }
#endif
constexpr uint32_t kNoThr = 0xFFFFFFFFu;
constexpr uint32_t kSpecial = 0x80000000u;  // entry is a nested block or a list
constexpr uint32_t kList = 0x40000000u;     // special entry is a short sorted list
constexpr uint32_t kIdxMask = 0x3FFFu;      // bucket index field (<= 8193 buckets)
constexpr uint32_t kSubShift = 14;          // packed sub-bucket field: bits 14..20
constexpr uint32_t kSubMask = 0x7Fu;
constexpr uint32_t kSubMax = 127;           // sub-buckets per group side that can be packed
constexpr uint32_t kIncShift = 21;          // sub-bucket increment flags of the 3 thresholds
constexpr uint32_t kRecMask = 0x3FFFFFFFu;  // level-1 boundary cell: record index

// Level-1 cell formats (per column, chosen by the planner):
enum LutFmt : uint8_t {
    FMT32 = 0,   // u32: plain = idx (0..13) | sub (14..20); boundary = kSpecial | record index
    FMT16 = 1,   // u16: plain = idx (0..8) | sub (9..14);   boundary = 0x8000 | record index (15 bits)
    FMTEX = 2,   // u32, one cell per key value (s1 = 0, never a boundary): idx (0..8) | sub (9..14) |
                 //      HLL register index (15..26) | HLL rank (27..31) of that key (int32 columns)
    FMT1T = 3,   // u32 with one in-cell threshold (specialised kernel only; 1 <= s1 <= 20):
                 //   bits [32-s1, 32): t = in-cell offset of the cell's breakpoint (0: none)
                 //   bit  31-s1      : special (>= 2 breakpoints): low bits = uint4 record index
                 //   bit  30-s1      : the breakpoint also cuts the packed sub-bucket
                 //   bits [0, 30-s1) : bs_lo = (bucket + 1) | sub << sb below the breakpoint
                 //   plain cell: t = 0 and bs_lo = bs - 1, so "offset >= t" always adds the 1 back.
                 // Decode: c = (u << (32-s1) | ones) >= e;  bs = c ? bs_lo + 1 + cut << sb : bs_lo.
                 // Buckets are 1-based in this format (the planner shifts the slot's histogram,
                 // grid and map addresses and its direct-pair intervals by one bucket).
};
constexpr uint32_t kRecMask16 = 0x7FFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;

#if defined(__CUDACC__)
#define GACE_HD __host__ __device__ __forceinline__
#else
#define GACE_HD inline
#endif

// Lookup table over the offset u = v - base of one column.  Level 1 is one u32 per cell
// of 2^s1 offsets:
//   plain    : bit 31 clear; bucket index (bits 0..13) | packed sub-bucket (bits 14..20) of
//              the whole cell (no breakpoint inside it) -- the common case: one LDS.32
//   boundary : kSpecial | uint4 index of the cell's 16-byte record:
//     direct : x = first bucket index (bits 0..13) | packed sub-bucket of that bucket
//              (bits 14..20) | flags (bits 21..23): threshold i also cuts the sub-buckets;
//              y <= z <= w = up to three thresholds (unused: ~0).
//              bucket = x.idx + #{t in (y, z, w) : u > t};  sub = x.sub + #{flagged t : u > t}
//     nested : x = kSpecial | sc << 24, y = uint4 index of a block of sub-records of size
//              2^sc; sub-record = R[y + ((u mod cell size) >> sc)] (any of the three kinds)
//     list   : x = kSpecial | kList | n << 24 | first bucket index, y = u32 index of n sorted
//              breakpoint offsets t; bucket = first + #{t : u >= t} (sub-bucket via the map)
//
// Packed sub-bucket of offset u from a DIRECT entry (kNone for a list entry).
GACE_HD uint32_t entry_sub(const uint4 &e, uint32_t u) {
    if (e.x & kSpecial) return kNone;
    return ((e.x >> kSubShift) & kSubMask) + ((u > e.y && (e.x >> kIncShift) & 1u) ? 1u : 0u) +
           ((u > e.z && (e.x >> (kIncShift + 1)) & 1u) ? 1u : 0u) + ((u > e.w && (e.x >> (kIncShift + 2)) & 1u) ? 1u : 0u);
}

// Final (direct or list) record reached from record `rec` of a cell of 2^s offsets.
template <class Mem>
GACE_HD uint4 rec_walk(const Mem &M, uint32_t rec, uint32_t s, uint32_t u) {
    uint4 e = M.u4(rec);
    while ((e.x & (kSpecial | kList)) == kSpecial) {        // block of sub-records (nested)
        const uint32_t sc = (e.x >> 24) & 63u;
        e = M.u4(e.y + ((u & ((1u << s) - 1u)) >> sc));
        s = sc;
    }
    return e;
}

// Final (direct or list) record for offset u, walking nested blocks (a plain cell is
// returned as a direct record without thresholds).  `M` reads the table image:
// M.u4(i) / M.u32(i) / M.u16(i) (shared memory in the kernel; a bounds-checked copy in
// gace_debug_buckets).  lut_w: u32 index of the level-1 table.
template <class Mem>
GACE_HD uint4 lut_entry(const Mem &M, uint32_t fmt, uint32_t lut_w, uint32_t s1, uint32_t u) {
    uint32_t rec;
    if (fmt == FMT16) {
        const uint32_t c = M.u16(2 * lut_w + (u >> s1));
        if (!(c & 0x8000u)) return make_uint4((c & 0x1FFu) | (((c >> 9) & 63u) << kSubShift), kNoThr, kNoThr, kNoThr);
        rec = c & kRecMask16;
    } else if (fmt == FMTEX) {
        const uint32_t c = M.u32(lut_w + u);
        return make_uint4((c & 0x1FFu) | (((c >> 9) & 63u) << kSubShift), kNoThr, kNoThr, kNoThr);
    } else {
        const uint32_t c = M.u32(lut_w + (u >> s1));
        if (!(c & kSpecial)) return make_uint4(c, kNoThr, kNoThr, kNoThr);
        rec = c & kRecMask;
    }
    return rec_walk(M, rec, s1, u);
}

// Bucket index of offset u from a final (direct or list) record.
template <class Mem>
GACE_HD uint32_t rec_bucket(const Mem &M, const uint4 &e, uint32_t u) {
    uint32_t b = e.x & kIdxMask;
    if (e.x & kList) {
        const uint32_t n = (e.x >> 24) & 63u;
        for (uint32_t i = 0; i < n; ++i) b += (u >= M.u32(e.y + i)) ? 1u : 0u;
        return b;
    }
    return b + (u > e.y ? 1u : 0u) + (u > e.z ? 1u : 0u) + (u > e.w ? 1u : 0u);
}

// FMT1T: field helpers (gace_plan.h LutFmt) and the bs = (bucket + 1) | sub << sb of offset u.
GACE_HD uint32_t t1_special(uint32_t s1) { return 1u << (31u - s1); }
GACE_HD uint32_t t1_dmask(uint32_t s1) { return (1u << (30u - s1)) - 1u; }
template <class Mem>
GACE_HD uint32_t t1_bs(const Mem &M, uint32_t lut_w, uint32_t s1, uint32_t sb, uint32_t u) {
    const uint32_t e = M.u32(lut_w + (u >> s1));
    if (e & t1_special(s1)) {                     // >= 2 breakpoints: walk the cell's record
        const uint4 r = rec_walk(M, e & t1_dmask(s1), s1, u);
        const uint32_t b = rec_bucket(M, r, u);
        const uint32_t sub = entry_sub(r, u);     // kNone for list records (caller maps it)
        return (b + 1u) | (sub == kNone ? 0u : sub << sb) | (sub == kNone ? 0x80000000u : 0u);
    }
    const uint32_t t = e >> (32u - s1), o = u & ((1u << s1) - 1u);
    const uint32_t lo = e & t1_dmask(s1), cut = (e >> (30u - s1)) & 1u;
    return o >= t ? lo + 1u + (cut << sb) : lo;
}

// Bucket index of offset u (full walk).
template <class Mem>
GACE_HD uint32_t lut_lookup(const Mem &M, uint32_t fmt, uint32_t lut_w, uint32_t s1, uint32_t u, uint32_t sb = 16) {
    if (fmt == FMT1T) return (t1_bs(M, lut_w, s1, sb, u) & ((1u << sb) - 1u)) - 1u;
    return rec_bucket(M, lut_entry(M, fmt, lut_w, s1, u), u);
}

enum SlotMode : uint8_t { MODE_LUT = 0, MODE_SEARCH = 1, MODE_NOPRED = 2 };

struct SlotParams {
    const void *ptr;        // device column base for this launch
    const int64_t *bps;     // MODE_SEARCH: sorted breakpoints (device)
    int64_t base;           // u = (uint32)(v - base)
    int64_t clamp_lo;       // clamped plans: v = min(max(v, clamp_lo), clamp_hi)
    int64_t clamp_hi;
    uint32_t nbp;           // MODE_SEARCH: number of breakpoints
    uint32_t s1;            // level-1 cell = u >> s1
    uint32_t lut_w;         // level-1 table: u32 index into shared memory
    uint32_t hist_addr;     // byte address of bucket 0 of this column's own histogram, or kNone
    uint32_t hll_idx;       // u32 index of this column's u32[4096] HLL registers, or kNone
    uint8_t dtype;          // 0 = int32, 1 = int64
    uint8_t mode;           // SlotMode
    uint8_t has_hll;
    int8_t prim_b;          // group whose sub-bucket this column's entries pack, or -1
    uint8_t fmt;            // LutFmt of the level-1 table
    uint8_t sb;             // sub-bucket shift inside bs (16, or the FMT1T bucket field width)
    uint8_t fdirect;        // exact cells holding the byte address of the key's own histogram bin
                            // (FMTEX, clamped, in no pair group): the bin add needs no arithmetic
    uint8_t pad;
    uint32_t bmask;         // (1 << sb) - 1: bucket field of bs
    uint32_t submask;       // sub-bucket field of bs >> sb (FMT16/FMTEX: 63, FMT32: 127)
    uint32_t sub_mul;       // 2^(32 - sb): bs >> sb as a high multiply (FMA pipe)
    uint32_t cell_mul;      // 2^(32 - s1) (s1 >= 1): level-1 cell u >> s1 as a high multiply
    // FMT1T decode constants (gace_plan.h LutFmt)
    uint32_t t1_mul;        // 2^(32 - s1)
    uint32_t t1_ones;       // 2^(32 - s1) - 1
    uint32_t t1_dmask;      // data bits
    uint32_t t1_sp;         // special flag
    uint32_t t1_cutsh;      // cut flag >> t1_cutsh lands on bit sb
    uint32_t t1_cutmul;     // 2^(32 - t1_cutsh), or 0 when t1_cutsh = 0
    // HLL by presence bitmap (small int32 domains): registers depend only on the set of
    // distinct kept values, so the scan records the set (one bit per value) and the
    // finalize hashes each present value once.  bm_addr = byte address of the CTA's bitmap
    // (kNone: u32 registers at hll_idx instead), bit i <-> value bm_base + i.
    uint32_t bm_addr;
    uint32_t bm_words;
    uint32_t bm_goff;       // word offset of this column's merged bitmap in g_bm
    uint32_t hll_out;       // output register block (ascending HLL column order)
    uint32_t bm_nvals;      // values in the column domain: the merged bitmap is complete at this count
    uint32_t hceil_off;     // byte offset of the column's register ceilings in g_hceil, or kNone
    // folded addressing (specialised kernels, int32 lookup columns whose cells are aligned
    // key multiples): level-1 byte address = (key >> s1) * 4 + fold_b; FMT1T in-cell offset
    // compare word = key * t1_mul + fold_z
    uint32_t fold_b;
    uint32_t fold_z;
    int64_t bm_base;        // multiple of 32
};

struct GroupParams {
    uint32_t grid_addr;     // byte address of grid[0][0]; grid[i][j] at + 4 * (i * nbs + j)
    uint32_t nbs;           // sub-buckets on the B side
    uint32_t map_addr;      // byte address of the B column's bucket -> sub-bucket map (u32 each)
    uint16_t dbeg, dend;    // this column pair's per-row ("direct") pairs: direct[dbeg .. dend)
    uint8_t a, b;           // slots: a = full-resolution side, b = sub-bucket side
    uint8_t has_grid;       // 2-D grid in shared memory (else all its pairs are direct)
    uint8_t packed;         // b's lookup-table entries carry this group's sub-bucket
};

// Cross-column pair evaluated per row (fallback when a group's grid does not fit).
struct DirectPair {
    uint32_t la, ha;        // bucket-index interval of the predicate on slot a (la > ha: empty)
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
    uint8_t *g_hll_part;                   // [CTA][hll_bytes] per-CTA register partials
    unsigned long long *g_nsamp;
    uint32_t *g_bm;                        // merged presence bitmaps (OR over CTAs; zeroed per probe)
    uint32_t *g_bmcnt;                     // [kMaxSlots] bits set in each merged bitmap (zeroed per probe)
    const uint8_t *g_hceil;                // per-column HLL register ceilings (max rank over the domain)
    uint32_t *g_hll_glob;                  // u32[hll_bytes]: registers merged across CTAs while the
                                           // scan runs (max; zeroed per probe) -> HLL skip bound
    uint64_t nrows;                        // rows in this launch
    uint64_t row0;                         // global id of the launch's first row
    uint64_t thr;                          // floor(rate * 2^64)
    uint64_t seed;
    uint32_t sample_all;                   // rate == 1
    uint32_t part_merge;                   // 1: max-merge into existing per-CTA partials (later chunk launches)
    uint32_t clamp;                        // clamp keys into each slot's [clamp_lo, clamp_hi]
    uint32_t c1, c4, c_hll;                // 1, 4, 2^p: multipliers the compiler cannot see, so that
                                           // u * 4 + base etc. stay IMADs (FMA pipe) instead of LEA/SHF
    uint32_t compact;                      // sampled launch: queue kept rows per warp (rate < 1/8)
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

// A column's bucket-count prefix: P(b) = g_pre[pre + b * stride] = #{kept rows with bucket < b}
// (own histogram: its exclusive prefix, stride 1; A side of a grid: the grid's summed-area
// table at the last column, stride nbs + 1).
struct FinPred {
    uint32_t pre, stride;
    uint32_t lo, hi;        // bucket interval (lo > hi: empty)
    uint32_t neg;
};

struct FinPair {
    uint32_t kind;
    uint32_t pre, stride;   // SAME: the column's prefix; GRID: SAT (row stride nb + 1); DIRECT: g_acc index
    uint32_t na, nb;        // GRID: grid extent
    uint32_t li, hi, lj, hj;// SAME: bucket intervals; GRID: i on the A side (buckets), j on the B side (sub-buckets)
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
    uint4 *zero;                // fin_output zeroes zero[0, zero_vec): the next call's accumulators
    uint64_t zero_vec;
    // presence-bitmap HLL columns: registers from the merged bitmap (fin_bitmap_hll)
    uint32_t nbm;
    const uint32_t *g_bm;
    struct BmJob {
        uint32_t goff, words, out, is64;
        int64_t base;
    } bm[kMaxSlots];
};

}  // namespace gace
