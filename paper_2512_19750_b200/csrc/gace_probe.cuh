// gace_probe.cuh -- device code of the probe kernel.
//
// Compiled twice:
//   * offline by nvcc into generic kernels probe_kernel<NC, SAMPLE, I64> (RtShape):
//     per-column / per-pair decisions are read from the kernel parameters at run time;
//   * at run time by NVRTC with a generated JitShape (gace_jit.cpp): the plan's shape --
//     column modes, dtypes, HLL flags, the list of column pairs -- is compile-time, so
//     the hot loop carries only the work this probe batch needs.
// Both instantiate the same probe_body<Shape>, so they compute the same bits.
//
// Per row unit (4*U rows per thread): 128-bit non-allocating loads of every probed
// column, prefetched one unit ahead; sample bits from SplitMix64 of the global row id;
// bucket ids from the shared-memory lookup tables (all level-1 reads issued before any is
// used, one branch for the rare nested / list / search entries); u32 bucket histograms
// (ATOMS.ADD); HLL: hash every key, touch shared memory only when the rank beats an exact
// per-warp lower bound of the registers (ATOMS.MAX); one 2-D grid bin per row and column
// pair; per-row evaluation for pairs whose grid did not fit.
#pragma once
#include "gace_plan.h"

#ifndef GACE_PREFETCH
#define GACE_PREFETCH 0
#endif
#ifndef GACE_L2_PF_DIST
#define GACE_L2_PF_DIST 2      // L2 prefetch distance in grid-stride iterations
#endif
// L2 prefetch of the column-streamed keys two iterations ahead: 0 none; 1 one PREFETCH per
// column; 2 one per iteration for int32 plans (lane-distributed), per column for int64 plans;
// 3 (default) none for int32 plans, per column for int64 plans -- measured (tools/variants.sh,
// GACE_JIT_DEFS=GACE_L2_PREFETCH=n): C5 1.95-1.96 ms without, 1.98 with; C5_i64 2.76 ms with,
// 3.12 without
#ifndef GACE_L2_PREFETCH
#define GACE_L2_PREFETCH 3
#endif
#ifndef GACE_L2_PREFETCH_U           // the same for the multi-quad units of 1-2 column probes
#define GACE_L2_PREFETCH_U 0
#endif
// GACE_CHECK=1 (specialised kernels: GACE_JIT_DEFS=GACE_CHECK=1): every shared-memory access
// through the helpers below is bounds-checked against the launch's dynamic shared memory and
// traps when outside it -- our own memcheck, since compute-sanitizer is closed on the B200 pool.
#ifndef GACE_CHECK
#define GACE_CHECK 0
#endif

namespace gace {

#define GACE_GAMMA 0x9E3779B97F4A7C15ULL

template <bool B, class T, class F> struct Cond { using type = T; };
template <class T, class F> struct Cond<false, T, F> { using type = F; };

// SplitMix64 finaliser (sample bit; int64 HLL hash).  DESIGN.md §2 steps 1 and 6.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// MurmurHash3 fmix32 (int32 HLL hash).  DESIGN.md §2 step 6.
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6BU;
    h ^= h >> 13;
    h *= 0xC2B2AE35U;
    h ^= h >> 16;
    return h;
}

__device__ __forceinline__ int4 ld_stream(const void *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

extern __shared__ uint4 g_smem[];

__device__ __forceinline__ void smem_check(uint32_t off, uint32_t bytes) {
    if (GACE_CHECK) {
        uint32_t dyn;
        asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        if (off > dyn || bytes > dyn - off) __trap();
    }
}

__device__ __forceinline__ uint32_t *smem32() { return reinterpret_cast<uint32_t *>(g_smem); }

// u32 in shared memory at byte address a (bucket counters, maps and grids are addressed
// in bytes so the hot loop never scales an index).
__device__ __forceinline__ uint32_t *at(uint32_t a) {
    smem_check(a, 4);
    return reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(g_smem) + a);
}

// Hot-path shared-memory accesses by byte offset from the dynamic shared memory: the
// window base is a uniform value the compiler folds into the address operand
// (LDS [R + UR]), instead of materialising generic pointers per access.
// (the address of the dynamic window taken from its PTX symbol: the compiler keeps it in a
// uniform register instead of re-deriving it from SR_CgaCtaId at every use; C5 scan -3 %)
__device__ __forceinline__ uint32_t sbase() { uint32_t v; asm("mov.u32 %0, _ZN4gace6g_smemE;" : "=r"(v)); return v; }
__device__ __forceinline__ uint32_t lds_u32(uint32_t off) {
    smem_check(off, 4);
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase() + off));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t off) {
    smem_check(off, 2);
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(sbase() + off));
    return v;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t off) {     // one LDS.128 (a record)
    smem_check(off, 16);
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(sbase() + off));
    return v;
}
__device__ __forceinline__ void red_add1(uint32_t off) {
    smem_check(off, 4);
    asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(sbase() + off) : "memory");
}

// Predicated shared-memory ops as single instructions (a C++ `if` around them becomes a
// branch with reconvergence barriers on every key).
__device__ __forceinline__ uint32_t saddr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// by byte offset into the dynamic window (the uniform base folds into the address operand)
__device__ __forceinline__ void red_max_if_off(bool pred, uint32_t off, uint32_t v) {
    if (pred) smem_check(off, 4);
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q red.shared.max.u32 [%1], %2;\n}"
                 :: "r"((uint32_t)pred), "r"(sbase() + off), "r"(v) : "memory");
}
__device__ __forceinline__ void red_max_if(bool pred, const uint32_t *addr, uint32_t v) {
    if (pred) smem_check(saddr(addr) - sbase(), 4);
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q red.shared.max.u32 [%1], %2;\n}"
                 :: "r"((uint32_t)pred), "r"(saddr(addr)), "r"(v) : "memory");
}
__device__ __forceinline__ void lds128_if(bool pred, const uint4 *addr, uint4 &r) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n @q ld.shared.v4.u32 {%0, %1, %2, %3}, [%5];\n}"
                 : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
                 : "r"((uint32_t)pred), "r"(saddr(addr)));
}

// Lower bound L of the FINAL registers of HLL column slot s (whole warp active).  The
// CTAs merge their registers into g_hll_glob (max) while the scan runs: this warp pulls
// its 1/nwarps slice of the merged registers, pushes the CTA's own values where they are
// higher, and records the slice minimum in s_slmin; L = min over the slice minima.  The
// merged registers only grow and every value in them came from some CTA's own rows, so a
// key whose rank is <= L cannot change the final max: skipping it is exact.
__shared__ uint8_t s_slmin[kMaxSlots][kThreads / 32];   // register values are < 64
__shared__ uint8_t s_slfull[kMaxSlots][kThreads / 32];  // warp slice reached the register ceilings
// Per-warp skip limit ~0 >> L (bit 0 cleared) of each HLL slot; row kThreads/32 stays ~1
// (no skipping) for the tail rows.  Kept in shared memory (a broadcast load per use)
// rather than in registers, which the hot loop needs for its keys.
__shared__ uint32_t s_wlim[kThreads / 32 + 1][kMaxSlots];

// Returns L | complete << 8: complete when ceil != nullptr and every warp's last slice check
// found the merged registers at their ceilings (the largest rank any domain value can
// give; registers only grow, so a slice once complete stays complete).
__device__ __noinline__ uint32_t hll_bound(uint32_t hll_idx, uint32_t *G, int s, const uint8_t *ceil) {
    // this warp's registers: i = warp * 32 + lane + j * kThreads (the warps cover all 4096)
    constexpr uint32_t kNw = kThreads / 32, kPer = (kHllM + kThreads - 1) / kThreads;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t i0 = warp * 32 + lane;
    const uint32_t *R = smem32() + hll_idx;
    uint32_t glob[kPer];
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j)                  // all loads in flight at once
        glob[j] = i0 + j * kThreads < kHllM ? __ldcg(G + i0 + j * kThreads) : 0xFFFFFFFFu;
    uint32_t m = 0xFFFFFFFFu;
    bool below = false;
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j) {
        const uint32_t i = i0 + j * kThreads;
        if (i >= kHllM) break;
        const uint32_t mine = R[i];
        if (mine > glob[j]) atomicMax(G + i, mine);
        const uint32_t merged = max(mine, glob[j]);
        m = min(m, merged);
        if (ceil && merged < __ldg(ceil + i)) below = true;
    }
    m = __reduce_min_sync(0xFFFFFFFFu, m);
    const bool slice_full = ceil != nullptr && !__any_sync(0xFFFFFFFFu, below);
    if (lane == 0) {
        s_slmin[s][warp] = (uint8_t)min(m, 255u);
        s_slfull[s][warp] = slice_full ? 1 : 0;
    }
    __syncwarp();
    uint32_t L = lane < kNw ? *reinterpret_cast<volatile uint8_t *>(&s_slmin[s][lane]) : 0xFFFFFFFFu;
    const bool f = lane < kNw ? *reinterpret_cast<volatile uint8_t *>(&s_slfull[s][lane]) != 0 : true;
    const bool complete = ceil != nullptr && __all_sync(0xFFFFFFFFu, f);
    return min(__reduce_min_sync(0xFFFFFFFFu, L), 255u) | (complete ? 256u : 0u);
}

// Bitmaps of at most this many words are pushed into the merged bitmap at the refresh points
// (so a domain the scan covers completely stops costing work early, C4); larger ones (C3's
// 2^20-value Zipf domain: 32K words, never complete) only at the CTA's end.
constexpr uint32_t kBmRefreshWords = 4096;

// Presence-bitmap slot s: this warp ORs its 1/nwarps slice of the CTA's bitmap into the
// merged bitmap g_bm, counting the bits it sets there for the first time, and reports
// whether the merged bitmap now holds every value of the column domain.  The registers
// depend only on the union of the bitmaps, so once it is complete no row can change the
// result and the CTAs stop testing keys (exact; C4: after the first ~8 iterations).
__device__ __noinline__ bool bm_push(const uint32_t *src, uint32_t *dst, uint32_t words, uint32_t *cnt,
                                     uint32_t nvals) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t fresh = 0;
    for (uint32_t i = warp * 32 + lane; i < words; i += kThreads) {
        const uint32_t w = *reinterpret_cast<const volatile uint32_t *>(src + i);
        if (w) fresh += __popc(w & ~atomicOr(dst + i, w));
    }
    fresh = __reduce_add_sync(0xFFFFFFFFu, fresh);
    uint32_t total = 0;
    if (lane == 0) total = fresh ? atomicAdd(cnt, fresh) + fresh : __ldcg(cnt);
    total = __shfl_sync(0xFFFFFFFFu, total, 0);
    return nvals && total >= nvals;
}

// #{t in bps : t <= v}, branch-free binary search (MODE_SEARCH fallback; out of line).
__device__ __noinline__ uint32_t search_bucket(const int64_t *bps, uint32_t n, int64_t v) {
    uint32_t lo = 0;
    while (n > 0) {
        const uint32_t half = n >> 1;
        const bool right = __ldg(bps + lo + half) <= v;
        lo = right ? lo + half + 1 : lo;
        n = right ? n - half - 1 : half;
    }
    return lo;
}

struct SmemTables {
    __device__ __forceinline__ uint4 u4(uint32_t i) const { smem_check(16 * i, 16); return g_smem[i]; }
    __device__ __forceinline__ uint32_t u32(uint32_t i) const { smem_check(4 * i, 4); return smem32()[i]; }
    __device__ __forceinline__ uint32_t u16(uint32_t i) const {
        smem_check(2 * i, 2);
        return reinterpret_cast<const uint16_t *>(g_smem)[i];
    }
};

// Full walk through nested cells and lists (out of line: rare special entries only).
__device__ __noinline__ uint32_t lut_bucket(uint32_t fmt, uint32_t lut_w, uint32_t s1, uint32_t u) {
    return lut_lookup(SmemTables{}, fmt, lut_w, s1, u);
}

__device__ __forceinline__ bool keep_row(const ProbeParams &P, uint64_t g) {
    return mix64(P.seed + (g + 1) * GACE_GAMMA) < P.thr;
}

// ------------------------------------------------------------------ plan shapes

// Plan layout read from the kernel parameters (shared-memory offsets, shifts, masks,
// multipliers): the generic kernels and the structure-keyed specialised kernels use it, so
// a new batch with the same plan structure reuses the compiled kernel; the layout-keyed
// variant (GACE_JIT_LAYOUT=1, design comparisons) bakes these in as immediates instead.
struct RtLayout {
    __device__ static uint32_t dbg(const ProbeParams &P) { return P.dbg; }
    __device__ static int64_t base(const ProbeParams &P, int s) { return P.slot[s].base; }
    __device__ static int64_t clo(const ProbeParams &P, int s) { return P.slot[s].clamp_lo; }
    __device__ static int64_t chi(const ProbeParams &P, int s) { return P.slot[s].clamp_hi; }
    __device__ static uint32_t s1(const ProbeParams &P, int s) { return P.slot[s].s1; }
    __device__ static uint32_t lutb(const ProbeParams &P, int s) { return 4 * P.slot[s].lut_w; }
    __device__ static uint32_t histb(const ProbeParams &P, int s) { return P.slot[s].hist_addr; }
    __device__ static uint32_t hllw(const ProbeParams &P, int s) { return P.slot[s].hll_idx; }
    __device__ static uint32_t bmaddr(const ProbeParams &P, int s) { return P.slot[s].bm_addr; }
    __device__ static uint32_t bmbase(const ProbeParams &P, int s) { return (uint32_t)P.slot[s].bm_base; }
    __device__ static uint32_t bmnv(const ProbeParams &P, int s) { return P.slot[s].bm_nvals; }
    __device__ static uint32_t hllout(const ProbeParams &P, int s) { return P.slot[s].hll_out; }
    __device__ static uint32_t sb(const ProbeParams &P, int s) { return P.slot[s].sb; }
    __device__ static uint32_t bmask(const ProbeParams &P, int s) { return P.slot[s].bmask; }
    __device__ static uint32_t t1mul(const ProbeParams &P, int s) { return P.slot[s].t1_mul; }
    __device__ static uint32_t t1ones(const ProbeParams &P, int s) { return P.slot[s].t1_ones; }
    __device__ static uint32_t t1dmask(const ProbeParams &P, int s) { return P.slot[s].t1_dmask; }
    __device__ static uint32_t t1sp(const ProbeParams &P, int s) { return P.slot[s].t1_sp; }
    __device__ static uint32_t t1cutsh(const ProbeParams &P, int s) { return P.slot[s].t1_cutsh; }
    __device__ static uint32_t t1cutmul(const ProbeParams &P, int s) { return P.slot[s].t1_cutmul; }
    __device__ static uint32_t submask(const ProbeParams &P, int s) { return P.slot[s].submask; }
    __device__ static uint32_t submul(const ProbeParams &P, int s) { return P.slot[s].sub_mul; }
    __device__ static uint32_t cellmul(const ProbeParams &P, int s) { return P.slot[s].cell_mul; }
    __device__ static uint32_t foldb(const ProbeParams &P, int s) { return P.slot[s].fold_b; }
    __device__ static uint32_t foldz(const ProbeParams &P, int s) { return P.slot[s].fold_z; }
    __device__ static uint32_t mapb(const ProbeParams &P, int s) {      // packed group's map, or kNone
        return P.slot[s].prim_b >= 0 ? P.grp[P.slot[s].prim_b].map_addr : kNone;
    }
    __device__ static uint32_t ggridb(const ProbeParams &P, int g) { return P.grp[g].grid_addr; }
    __device__ static uint32_t gnbs(const ProbeParams &P, int g) { return P.grp[g].nbs; }
    __device__ static uint32_t gmapb(const ProbeParams &P, int g) { return P.grp[g].map_addr; }
};

// Generic shape: only NC / SAMPLE / I64 are compile-time.
template <int NC_, bool SAMPLE_, bool I64_>
struct RtShape : RtLayout {
    static constexpr int NC = NC_;
    static constexpr bool SAMPLE = SAMPLE_;
    static constexpr bool I64 = I64_;
    static constexpr bool STATIC = false;
    static constexpr bool ANY_HLL = true;          // refresh points always present
    static constexpr int U = NC >= 4 ? 1 : 4 / NC;
    static constexpr int NG = 0;
    __device__ static bool active(const ProbeParams &P, int s) { return s < (int)P.nslots; }
    __device__ static int mode(const ProbeParams &P, int s) { return P.slot[s].mode; }
    __device__ static bool is32(const ProbeParams &P, int s) { return !I64 || P.slot[s].dtype == 0; }
    __device__ static bool hll(const ProbeParams &P, int s) { return P.slot[s].has_hll; }
    __device__ static bool clamp(const ProbeParams &P) { return P.clamp; }
    __device__ static bool packs(const ProbeParams &P, int s) { return P.slot[s].prim_b >= 0; }
    __device__ static bool ownh(const ProbeParams &P, int s) {
        return P.slot[s].mode != MODE_NOPRED && P.slot[s].hist_addr != kNone;
    }
    __device__ static bool fdirect(const ProbeParams &P, int s) { return P.slot[s].fdirect != 0; }
    __device__ static constexpr bool gpacked(int) { return false; }
    __device__ static constexpr bool clust(const ProbeParams &, int) { return false; }
    __device__ static int fmt(const ProbeParams &P, int s) { return P.slot[s].fmt; }
    __device__ static constexpr int ga(int) { return 0; }
    __device__ static constexpr int gb(int) { return 0; }
    __device__ static constexpr bool ggrid(int) { return false; }
    __device__ static constexpr bool gdirect(int) { return false; }
    __device__ static bool sclamp(const ProbeParams &P, int) { return P.clamp; }
    __device__ static bool hllbm(const ProbeParams &P, int s) { return P.slot[s].bm_addr != kNone; }
    __device__ static constexpr bool fold(const ProbeParams &, int) { return false; }
};

// ------------------------------------------------------------------ row units

template <class Sh>
using KeyT = typename Cond<Sh::I64, int64_t, int32_t>::type;

template <class Sh>
struct Unit {
    int4 r[Sh::NC][Sh::U][Sh::I64 ? 2 : 1];
};

template <class Sh>
__device__ __forceinline__ void load_unit(const ProbeParams &P, uint32_t u, Unit<Sh> &X) {
#pragma unroll
    for (int s = 0; s < Sh::NC; ++s) {
        if (!Sh::active(P, s)) continue;
        const char *base = static_cast<const char *>(P.slot[s].ptr);
        if (Sh::is32(P, s)) {
#pragma unroll
            for (int j = 0; j < Sh::U; ++j) X.r[s][j][0] = ld_stream(base + ((uint64_t)u * Sh::U + j) * 16);
        } else {
#pragma unroll
            for (int j = 0; j < Sh::U; ++j) {
                X.r[s][j][0] = ld_stream(base + ((uint64_t)u * Sh::U + j) * 32);
                X.r[s][j][Sh::I64 ? 1 : 0] = ld_stream(base + ((uint64_t)u * Sh::U + j) * 32 + 16);
            }
        }
    }
}

// Column s of unit u (U == 1 layout) into r.
template <class Sh>
__device__ __forceinline__ void load_col(const ProbeParams &P, int s, uint32_t u, int4 (&r)[Sh::I64 ? 2 : 1]) {
    const char *base = static_cast<const char *>(P.slot[s].ptr);
    if (Sh::is32(P, s)) {
        r[0] = ld_stream(base + (uint64_t)u * 16);
    } else {
        r[0] = ld_stream(base + (uint64_t)u * 32);
        r[Sh::I64 ? 1 : 0] = ld_stream(base + (uint64_t)u * 32 + 16);
    }
}

template <class Sh>
__device__ __forceinline__ void decode(const ProbeParams &P, int s, const int4 (&r)[Sh::I64 ? 2 : 1],
                                       KeyT<Sh> (&v)[4]) {
    if (Sh::is32(P, s)) {
        v[0] = r[0].x; v[1] = r[0].y; v[2] = r[0].z; v[3] = r[0].w;
    } else {
        const int4 &a = r[0], &b = r[Sh::I64 ? 1 : 0];
        v[0] = static_cast<KeyT<Sh>>((static_cast<int64_t>(a.y) << 32) | static_cast<uint32_t>(a.x));
        v[1] = static_cast<KeyT<Sh>>((static_cast<int64_t>(a.w) << 32) | static_cast<uint32_t>(a.z));
        v[2] = static_cast<KeyT<Sh>>((static_cast<int64_t>(b.y) << 32) | static_cast<uint32_t>(b.x));
        v[3] = static_cast<KeyT<Sh>>((static_cast<int64_t>(b.w) << 32) | static_cast<uint32_t>(b.z));
    }
}

// Offset u = key - base of a lookup-table column (with the optional clamp).
template <class Sh>
__device__ __forceinline__ uint32_t offset_of(const ProbeParams &P, int s, KeyT<Sh> xk) {
    if (Sh::is32(P, s)) {
        int32_t y = static_cast<int32_t>(xk);
        if (Sh::sclamp(P, s))
            y = min(max(y, static_cast<int32_t>(Sh::clo(P, s))), static_cast<int32_t>(Sh::chi(P, s)));
        return static_cast<uint32_t>(y) - static_cast<uint32_t>(Sh::base(P, s));
    }
    int64_t x = xk;
    if (Sh::sclamp(P, s)) x = min(max(x, Sh::clo(P, s)), Sh::chi(P, s));
    return static_cast<uint32_t>(static_cast<uint64_t>(x) - static_cast<uint64_t>(Sh::base(P, s)));
}

// Bucket | sub-bucket << 16 of a key in a boundary cell: its 16-byte record (<= 3
// thresholds), or the full walk for nested / list records (sub-bucket via the map).
template <class Sh>
__device__ __forceinline__ uint32_t boundary_bucket(const ProbeParams &P, int s, uint32_t rec, uint32_t u) {
    const uint4 r = lds_u4(16 * rec);
    if (!(r.x & kSpecial)) {
        const uint32_t c1 = u > r.y, c2 = u > r.z, c3 = u > r.w;
        uint32_t b = (r.x & kIdxMask) + c1 + c2 + c3;
        if (Sh::packs(P, s))
            b |= (((r.x >> kSubShift) & kSubMask) + (c1 & (r.x >> kIncShift)) + (c2 & (r.x >> (kIncShift + 1))) +
                  (c3 & (r.x >> (kIncShift + 2)))) << Sh::sb(P, s);
        return b;
    }
    const uint32_t b = lut_bucket(Sh::fmt(P, s), Sh::lutb(P, s) / 4, Sh::s1(P, s), u);
    return b | (Sh::packs(P, s) ? *at(Sh::mapb(P, s) + 4 * b) << Sh::sb(P, s) : 0u);
}

// FMT1T cell with >= 2 breakpoints: bs = (bucket + 1) | sub << sb from its record (out of
// line; list records take the sub-bucket from the packed group's map).
// (Arguments by value: a reference to the kernel parameters would turn every field read
// in the callee into a generic-memory load.)
__device__ __noinline__ uint32_t t1_special_bs(uint32_t lut_w, uint32_t s1, uint32_t sb, uint32_t map_addr,
                                               uint32_t u) {
    const uint32_t v = t1_bs(SmemTables{}, lut_w, s1, sb, u);
    if (!(v & 0x80000000u)) return v;
    const uint32_t b1 = v & ((1u << sb) - 1u);
    return b1 | (map_addr != kNone ? *at(map_addr + 4 * b1) << sb : 0u);
}

// bs = bucket | sub-bucket << sb of slot s over one row quad (the layout of the slot's plain
// level-1 word, so a plain cell is used as is; FMT1T buckets are 1-based).  One LDS per key
// (one per quad for a clustered column whose four keys are equal); cells with breakpoints
// resolve inline (FMT1T: one threshold) or, for the rare special cells, through one test
// per column quad and a record walk.  Multiplies by 2^k use opaque multipliers (P.c4,
// P.slot[].t1_mul) or high multiplies so that they run on the FMA pipe.
template <class Sh, int NK>
__device__ __forceinline__ void bucket_col(const ProbeParams &P, int s, const KeyT<Sh> (&v)[4],
                                           uint32_t (&bs)[4], uint32_t (&e)[4]) {
    const bool lut = Sh::active(P, s) && Sh::mode(P, s) == MODE_LUT;
    const uint32_t base = Sh::lutb(P, s);
    const int f = Sh::fmt(P, s);
    constexpr int nk = NK;
    constexpr bool same = NK == 1;
    uint32_t u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        u[k] = 0u;
        e[k] = 0u;
        if (k >= nk || !lut) continue;
        if (Sh::fold(P, s)) {          // base folded into the immediates: index with the key itself
            const uint32_t x = static_cast<uint32_t>(v[k]);
            const uint32_t cell = f == FMTEX ? x : __umulhi(x, Sh::cellmul(P, s));
            e[k] = lds_u32(cell * P.c4 + Sh::foldb(P, s));
            continue;
        }
        u[k] = offset_of<Sh>(P, s, v[k]);
        if (f == FMT16) {
            const uint32_t cell = u[k] >> Sh::s1(P, s);
            e[k] = lds_u16(base + 2 * cell);
        } else {
            const uint32_t cell = f == FMTEX ? u[k] : (Sh::s1(P, s) ? __umulhi(u[k], Sh::cellmul(P, s)) : u[k]);
            e[k] = lds_u32(cell * P.c4 + base);
        }
    }
    if (lut && f == FMT1T) {           // one in-cell threshold: c ? lo + inc : lo, inc = 1 or 1 + 2^sb
        const uint32_t sp = Sh::t1sp(P, s);
        uint32_t any = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= nk) continue;
            const uint32_t x = e[k];
            const uint32_t zz = Sh::fold(P, s) ? static_cast<uint32_t>(v[k]) * P.slot[s].t1_mul + Sh::foldz(P, s)
                                               : u[k] * P.slot[s].t1_mul + Sh::t1ones(P, s);
            const uint32_t lo = x & Sh::t1dmask(P, s);
            uint32_t inc = 1u;
            if (Sh::packs(P, s))
                inc = ((Sh::t1cutsh(P, s) ? __umulhi(x, Sh::t1cutmul(P, s)) : x) & (Sh::bmask(P, s) + 1u)) | 1u;
            bs[k] = lo + (zz >= x ? inc : 0u);
            any |= x;
        }
        if (any & sp) {                // >= 2 breakpoints in some cell
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k >= nk || !(e[k] & sp)) continue;
                if (Sh::fold(P, s)) u[k] = offset_of<Sh>(P, s, v[k]);
                const uint4 r = lds_u4(16 * (e[k] & Sh::t1dmask(P, s)));
                if (!(r.x & kSpecial)) {   // direct record, <= 3 thresholds: inline
                    const uint32_t c1 = u[k] > r.y, c2 = u[k] > r.z, c3 = u[k] > r.w;
                    uint32_t b = (r.x & kIdxMask) + 1u + c1 + c2 + c3;
                    if (Sh::packs(P, s))
                        b |= (((r.x >> kSubShift) & kSubMask) + (c1 & (r.x >> kIncShift)) +
                              (c2 & (r.x >> (kIncShift + 1))) + (c3 & (r.x >> (kIncShift + 2)))) << Sh::sb(P, s);
                    bs[k] = b;
                } else {                   // nested block or list: out-of-line walk
                    bs[k] = t1_special_bs(Sh::lutb(P, s) / 4, Sh::s1(P, s), Sh::sb(P, s),
                                          Sh::packs(P, s) ? Sh::mapb(P, s) : kNone, u[k]);
                }
            }
        }
    } else if (lut && f == FMT32) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= nk) continue;
            bs[k] = e[k];
            if (e[k] & kSpecial) bs[k] = boundary_bucket<Sh>(P, s, e[k] & kRecMask, u[k]);
        }
    } else if (lut && f == FMT16) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= nk) continue;
            bs[k] = e[k];
            if (e[k] & 0x8000u) bs[k] = boundary_bucket<Sh>(P, s, e[k] & kRecMask16, u[k]);
        }
    } else if (lut) {                  // FMTEX: exact cells, never a boundary
#pragma unroll
        for (int k = 0; k < 4; ++k) bs[k] = e[k];
    } else if (Sh::active(P, s) && Sh::mode(P, s) == MODE_SEARCH) {      // binary-search fallback column
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= nk) continue;
            const uint32_t b = search_bucket(P.slot[s].bps, P.slot[s].nbp, v[k]);
            bs[k] = b | (Sh::packs(P, s) ? *at(Sh::mapb(P, s) + 4 * b) << 16 : 0u);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) bs[k] = 0u;
    }
    if (same) {
        bs[1] = bs[2] = bs[3] = bs[0];
        e[1] = e[2] = e[3] = e[0];
    }
}

__device__ __forceinline__ void direct_pairs(const ProbeParams &P, uint32_t ma, uint32_t mb, const GroupParams &G,
                                             const uint32_t (&bsa)[4], const uint32_t (&bsb)[4], uint32_t keep) {
    for (uint32_t d = G.dbeg; d < G.dend; ++d) {
        const DirectPair D = P.direct[d];
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t ba = bsa[k] & ma, bb = bsb[k] & mb;
            const uint32_t ina = ((ba >= D.la) & (ba <= D.ha)) ^ D.nega;
            const uint32_t inb = ((bb >= D.lb) & (bb <= D.hb)) ^ D.negb;
            c += ((keep >> k) & 1u) & ina & inb;
        }
        // per-thread add: this may run in a diverged warp (sampled quads), where a
        // warp-collective reduction over __activemask() is not well defined
        if (c) atomicAdd(smem32() + D.acc_idx, c);
    }
}

// grid[bucket of a][sub-bucket of b] += 1 for each kept row (sub: packed or via the map)
__device__ __forceinline__ void grid_add(uint32_t c4, uint32_t amask, uint32_t bsh, uint32_t submask, uint32_t bmask,
                                         uint32_t grid, uint32_t nbs, uint32_t map, bool packed,
                                         const uint32_t (&bsa)[4], const uint32_t (&bsb)[4], uint32_t keep) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if ((keep >> k) & 1u) {
            const uint32_t sub = packed ? (bsb[k] >> bsh) & submask : *at(map + 4 * (bsb[k] & bmask));
            red_add1(((bsa[k] & amask) * nbs + sub) * c4 + grid);
        }
    }
}

template <int NC>
__device__ __forceinline__ uint32_t pick(const uint32_t (&x)[NC][4], uint32_t s, int k) {
    uint32_t r = x[0][k];
#pragma unroll
    for (int c = 1; c < NC; ++c) r = (s == (uint32_t)c) ? x[c][k] : r;
    return r;
}

// Own bucket histogram (columns that are no grid's full-resolution side) and HLL of one
// column of a row quad.
template <class Sh, int NK>
__device__ __forceinline__ void column_tail(const ProbeParams &P, int s, uint32_t keep, const uint32_t *wlim,
                                            uint32_t bmfull, const KeyT<Sh> (&v)[4], const uint32_t (&bs)[4],
                                            const uint32_t (&ex)[4]) {
    constexpr bool same = NK == 1;
    uint32_t *sm = smem32();
    const uint32_t dbg = Sh::dbg(P);
    if (Sh::ownh(P, s) && !(dbg & 2)) {
        const uint32_t h = Sh::histb(P, s);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((keep >> k) & 1u) red_add1(Sh::fdirect(P, s) ? bs[k] : h + 4 * (bs[k] & Sh::bmask(P, s)));
    }
    // HLL: w = (hash << p) | 2^(p-1), rank = clz(w) + 1; rank > lower bound L  <=>  w <= ~0 >> L.
    // Shifts by constants are written as multiplies (IMAD / IMAD.HI run on the FMA pipe,
    // which the rest of the loop leaves idle); survivors do a predicated ATOMS.MAX.
    if (Sh::hll(P, s) && Sh::hllbm(P, s) && !(dbg & 8)) {
        if ((bmfull >> s) & 1u) return;        // merged bitmap complete: nothing left to record
        // presence bitmap: set the bit of each kept value (test first: after the first rows
        // nearly every value is present, so the quad costs four loads and no atomics)
        uint32_t wa[4], bit[4], need = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t u = static_cast<uint32_t>(v[k]) - Sh::bmbase(P, s);
            wa[k] = (u >> 5) * P.c4 + Sh::bmaddr(P, s);
            bit[k] = 1u << (u & 31u);
            const bool kept_k = same ? keep != 0 : ((keep >> k) & 1u);
            if (kept_k && !(lds_u32(wa[k]) & bit[k])) need |= 1u << k;
            if (same) break;
        }
        if (need) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((need >> k) & 1u)
                    asm volatile("red.shared.or.b32 [%0], %1;" :: "r"(sbase() + wa[k]), "r"(bit[k]) : "memory");
        }
    } else if (Sh::hll(P, s) && !(dbg & 8)) {
        if ((bmfull >> s) & 1u) return;        // registers at their ceilings: nothing can change
        uint32_t *R = sm + Sh::hllw(P, s);
        if (Sh::mode(P, s) == MODE_LUT && Sh::fmt(P, s) == FMTEX && !Sh::sclamp(P, s)) {
            // (index, rank) precomputed per key value in its exact cell.  A CTA needs each
            // value's contribution once: the first thread to apply it clears the rank in the
            // cell (a benign race -- every writer stores the same word), so repeats of the
            // value skip the register entirely.  One test covers the quad.
            uint32_t any = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) any |= ((keep >> k) & 1u) ? ex[k] : 0u;
            if ((any >> 27) && !(dbg & 1)) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t x = ex[k], rank = x >> 27;
                    if (((keep >> k) & 1u) && rank) {
                        atomicMax(R + ((x >> 15) & 0xFFFu), rank);
                        *at(Sh::lutb(P, s) + 4 * offset_of<Sh>(P, s, v[k])) = x & 0x07FFFFFFu;
                    }
                }
            }
        } else if (Sh::is32(P, s)) {
            // w32 is even, so clearing bit 0 keeps "w32 <= lim" and puts the non-kept marker ~0 above it
            const uint32_t lim = wlim[s];
            uint32_t w32[4], idx[4], wmin = 0xFFFFFFFFu;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t h = static_cast<uint32_t>(v[k]);
                // fmix32; one shift on the FMA pipe (high multiply), two on the ALU pipe, so
                // the hash block does not pile onto one pipe (5 FMA + 5 ALU ops)
                h ^= h >> 16;
                h *= 0x85EBCA6BU;
                h ^= __umulhi(h, 1u << 19);
                h *= 0xC2B2AE35U;
                h ^= h >> 16;                                        // = fmix32(x)
                w32[k] = h * P.c_hll + (1u << (kHllP - 1));          // never ~0 (low bits 0x800)
                idx[k] = h >> (32 - kHllP);
                const bool kept_k = (same && k > 0) ? false : (same ? keep != 0 : ((keep >> k) & 1u));
                if (!kept_k) w32[k] = 0xFFFFFFFFu;
                wmin = min(wmin, w32[k]);
                if (same) break;
            }
            // one test for the quad: some key's rank beats the lower bound L
            if (wmin <= lim && !(dbg & 1)) {
                // exact test against the CTA's register first (all loads issued, then the
                // compares): a frequent value whose rank is already in (a skewed column's
                // head, e.g. fmix32(0) = 0 -> rank 21) never reaches the atomic
                // rank > cur  <=>  w <= ~0 >> cur (cur <= 21; 31 marks "not a survivor": w >= 2^11)
                // (registers addressed by byte offset from the dynamic window's uniform base)
                const uint32_t roff = 4 * Sh::hllw(P, s);
                uint32_t cur[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    cur[k] = w32[k] <= lim ? lds_u32(roff + 4 * idx[k]) : 31u;
                    if (same) break;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    red_max_if_off(w32[k] <= (0xFFFFFFFFu >> cur[k]), roff + 4 * idx[k], __clz(w32[k]) + 1);
                    if (same) break;
                }
            }
        } else {
            const uint64_t lim = ~0ull >> (32 - __popc(wlim[s] | 1u));     // L from the 32-bit limit
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t h = mix64(static_cast<uint64_t>(v[k]) + GACE_GAMMA);
                const uint64_t w64 = (h << kHllP) | (1ull << (kHllP - 1));
                const uint32_t idx = static_cast<uint32_t>(h >> (64 - kHllP));
                red_max_if(((keep >> k) & 1u) && w64 <= lim && !(dbg & 1), R + idx, __clzll(w64) + 1);
            }
        }
    }
}

// Pair grids / per-row pairs of one row quad.
template <class Sh>
__device__ __forceinline__ void pair_work(const ProbeParams &P, uint32_t keep, const uint32_t (&bs)[Sh::NC][4]) {
    constexpr int NC = Sh::NC;
    if (Sh::STATIC) {
#pragma unroll
        for (int g = 0; g < Sh::NG; ++g) {
            const GroupParams &G = P.grp[g];
            const int a = Sh::ga(g), b = Sh::gb(g);
            if (Sh::ggrid(g))
                grid_add(P.c4, Sh::bmask(P, a), Sh::sb(P, b), Sh::submask(P, b), Sh::bmask(P, b), Sh::ggridb(P, g),
                         Sh::gnbs(P, g), Sh::gmapb(P, g), Sh::gpacked(g), bs[a], bs[b], keep);
            if (Sh::gdirect(g)) direct_pairs(P, Sh::bmask(P, a), Sh::bmask(P, b), G, bs[a], bs[b], keep);
        }
    } else {
        for (uint32_t g = 0; g < P.ngroups; ++g) {
            const GroupParams &G = P.grp[g];
            uint32_t ba[4], bb[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                ba[k] = pick<NC>(bs, G.a, k);
                bb[k] = pick<NC>(bs, G.b, k);
            }
            if (G.has_grid)
                grid_add(P.c4, P.slot[G.a].bmask, P.slot[G.b].sb, P.slot[G.b].submask, P.slot[G.b].bmask,
                         G.grid_addr, G.nbs, G.map_addr, G.packed, ba, bb, keep);
            if (G.dend > G.dbeg) direct_pairs(P, P.slot[G.a].bmask, P.slot[G.b].bmask, G, ba, bb, keep);
        }
    }
}

// Everything one row quad contributes.  keep: one bit per row.
// unext != kNoUnit: once column s is consumed, its registers are refilled with column s of
// unit unext, so the next unit's keys are in flight during the rest of this one (no extra
// registers: a software pipeline column by column).
constexpr uint32_t kNoUnit = 0xFFFFFFFFu;
template <class Sh>
__device__ __forceinline__ void quad_work(const ProbeParams &P, int4 (&r)[Sh::NC][Sh::I64 ? 2 : 1],
                                          uint32_t keep, const uint32_t *wlim, uint32_t bmfull,
                                          uint32_t unext = kNoUnit) {
    constexpr int NC = Sh::NC;
    uint32_t *sm = smem32();
    const uint32_t dbg = Sh::dbg(P);
    uint32_t bs[NC][4];
    // one column at a time (bucket, own histogram, HLL): only that column's keys and lookup
    // words are live next to the quad's bucket words
#pragma unroll
    for (int s = 0; s < NC; ++s) {
        if (!Sh::active(P, s)) {
            bs[s][0] = bs[s][1] = bs[s][2] = bs[s][3] = 0u;
            continue;
        }
        KeyT<Sh> v[4];
        decode<Sh>(P, s, r[s], v);
        // clustered column, all four keys equal: one lookup and one hash cover the quad
        uint32_t ex[4];
        if (Sh::clust(P, s) && v[0] == v[1] && v[1] == v[2] && v[2] == v[3]) {
            bucket_col<Sh, 1>(P, s, v, bs[s], ex);
            column_tail<Sh, 1>(P, s, keep, wlim, bmfull, v, bs[s], ex);
        } else {
            bucket_col<Sh, 4>(P, s, v, bs[s], ex);
            column_tail<Sh, 4>(P, s, keep, wlim, bmfull, v, bs[s], ex);
        }
        if (unext != kNoUnit) load_col<Sh>(P, s, unext, r[s]);
    }
    // pairs
    if (dbg & 4) return;
    pair_work<Sh>(P, keep, bs);
}

// Row r of the launch alone (scalar loads of its keys, replicated over a quad whose rows
// 1..3 are masked off): the ragged tail, and the compacted rows of a sparse sample.
template <class Sh>
__device__ __forceinline__ void load_row(const ProbeParams &P, uint64_t r, int4 (&rj)[Sh::NC][Sh::I64 ? 2 : 1]) {
#pragma unroll
    for (int s = 0; s < Sh::NC; ++s) {
        if (!Sh::active(P, s)) continue;
        if (Sh::is32(P, s)) {
            const int32_t x = __ldg(static_cast<const int32_t *>(P.slot[s].ptr) + r);
            rj[s][0] = make_int4(x, x, x, x);     // rows 1..3 of the quad are masked off
        } else {
            const long long x = __ldg(static_cast<const long long *>(P.slot[s].ptr) + r);
            const int lo = (int)(x & 0xFFFFFFFF), hi = (int)(x >> 32);
            rj[s][0] = make_int4(lo, hi, lo, hi);
            rj[s][Sh::I64 ? 1 : 0] = make_int4(lo, hi, lo, hi);
        }
    }
}

// One row past the last full unit (out of line: cold code).
template <class Sh>
__device__ __noinline__ uint32_t tail_row(const ProbeParams &P, uint64_t r) {
    const uint32_t keep = (!Sh::SAMPLE || keep_row(P, P.row0 + r)) ? 1u : 0u;
    if (!keep) return 0;
    int4 rj[Sh::NC][Sh::I64 ? 2 : 1];
    load_row<Sh>(P, r, rj);
    quad_work<Sh>(P, rj, 1u, s_wlim[kThreads / 32], 0u);
    return 1;
}

// Sparse samples (rate < 3/8, gace_host.cpp P.compact): each warp hashes the sample bits of its row quads, queues the
// kept rows' indices in shared memory, and works on them 32 at a time -- every lane one kept
// row -- instead of running the per-quad work for the few lanes whose quad kept a row (at rate
// 0.01, 72 % of the warps had a kept row somewhere, so almost every warp paid the whole quad
// work at 1/32 of its lanes).  Only kept rows' keys are read.
constexpr uint32_t kQueue = 64;                       // entries per warp (ring)
__shared__ uint32_t s_queue[kThreads / 32][kQueue];
static_assert(sizeof(uint32_t) * (kThreads / 32) * kQueue + 2 * kMaxSlots * (kThreads / 32) +
                  4 * (kThreads / 32 + 1) * kMaxSlots <= kStaticSmem, "static shared memory over kStaticSmem");
static_assert(2 * kMaxSlots * (kThreads / 32) + 4 * (kThreads / 32 + 1) * kMaxSlots <= kStaticSmemFull,
              "a full scan's static shared memory over kStaticSmemFull");

template <class Sh>
__device__ __forceinline__ void probe_body(const ProbeParams &P) {
    constexpr int NC = Sh::NC, U = Sh::U;
    uint32_t *sm = smem32();
    // tables -> shared memory; accumulators and registers -> 0
    for (uint32_t i = threadIdx.x; i < P.image_u4; i += blockDim.x) g_smem[i] = __ldg(P.image + i);
    for (uint32_t i = P.image_u4 + threadIdx.x; i < P.smem_bytes / 16; i += blockDim.x)
        g_smem[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < kMaxSlots * (kThreads / 32)) (&s_slmin[0][0])[threadIdx.x] = 0;
    if (threadIdx.x < kMaxSlots * (kThreads / 32)) (&s_slfull[0][0])[threadIdx.x] = 0;
    if (threadIdx.x < kMaxSlots * (kThreads / 32 + 1)) (&s_wlim[0][0])[threadIdx.x] = 0xFFFFFFFEu;
    __syncthreads();

    // unit indices fit 32 bits: the host caps a launch at 2^31 units
    const uint32_t nunits = static_cast<uint32_t>(P.nrows / (4 * U));
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t kept = 0;
    uint32_t *wlim = s_wlim[threadIdx.x >> 5];
    uint32_t it = 0, next_refresh = 4;
    uint32_t bmfull = 0;       // bit s: slot s's HLL is complete -- merged presence bitmap full, or
                               // merged registers at their ceilings (warp-uniform)
    auto body = [&](const Unit<Sh> &X, uint32_t u) {
        if (Sh::ANY_HLL && it == next_refresh) {
            next_refresh = it + min(it, 32u);
            if (__activemask() == 0xFFFFFFFFu) {
#pragma unroll
                for (int s = 0; s < NC; ++s)
                    if (Sh::active(P, s) && Sh::hll(P, s) && !Sh::hllbm(P, s) && !((bmfull >> s) & 1u)) {
                        const uint32_t hc = P.slot[s].hceil_off;
                        const uint32_t hb = hll_bound(Sh::hllw(P, s), P.g_hll_glob + Sh::hllout(P, s) * kHllM, s,
                                                      hc != kNone ? P.g_hceil + hc : nullptr);
                        const uint32_t L = min(hb & 255u, 31u);
                        if ((threadIdx.x & 31) == 0) wlim[s] = (0xFFFFFFFFu >> L) & 0xFFFFFFFEu;
                        if (hb >> 8) bmfull |= 1u << s;       // registers at their ceilings: column complete
                    }
                    else if (Sh::active(P, s) && Sh::hll(P, s) && Sh::hllbm(P, s) && !((bmfull >> s) & 1u) &&
                             P.slot[s].bm_words <= kBmRefreshWords &&
                             bm_push(smem32() + Sh::bmaddr(P, s) / 4, P.g_bm + P.slot[s].bm_goff,
                                     P.slot[s].bm_words, P.g_bmcnt + s, Sh::bmnv(P, s)))
                        bmfull |= 1u << s;
                __syncwarp();
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t keep = 0xFu;
            if (Sh::SAMPLE) {
                const uint64_t g0 = P.row0 + ((uint64_t)u * U + j) * 4;
                keep = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) keep |= (keep_row(P, g0 + k) ? 1u : 0u) << k;
                kept += __popc(keep);
                if (!keep) continue;
            }
            int4 rj[NC][Sh::I64 ? 2 : 1];
#pragma unroll
            for (int s = 0; s < NC; ++s) {
                rj[s][0] = X.r[s][j][0];
                if (Sh::I64) rj[s][Sh::I64 ? 1 : 0] = X.r[s][j][Sh::I64 ? 1 : 0];
            }
            quad_work<Sh>(P, rj, keep, wlim, bmfull);
        }
        ++it;
    };
    uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    // sample bits of a row quad (all four rows when the probe is not sampled)
    auto quad_keep = [&](uint32_t uu) -> uint32_t {
        if (!Sh::SAMPLE) return 0xFu;
        // SplitMix64 states of consecutive rows differ by gamma: one 64-bit multiply per quad
        uint64_t z = P.seed + (P.row0 + (uint64_t)uu * 4 + 1) * GACE_GAMMA;
        uint32_t kk = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k, z += GACE_GAMMA) kk |= (mix64(z) < P.thr ? 1u : 0u) << k;
        return kk;
    };
    if (Sh::SAMPLE && P.compact) {
        const uint32_t lane = threadIdx.x & 31;
        uint32_t *q = s_queue[threadIdx.x >> 5];
        uint32_t qh = 0, qt = 0;                       // ring head / tail (warp-uniform)
        // kept rows of the queue head, one per lane (all 32 lanes, or the last partial batch)
        auto work = [&](uint32_t nb) {
            if (lane < nb) {
                int4 rj[NC][Sh::I64 ? 2 : 1];
                load_row<Sh>(P, q[(qh + lane) % kQueue], rj);
                quad_work<Sh>(P, rj, 1u, wlim, bmfull);
            }
            qh += nb;
            __syncwarp();
        };
        // row quads below the tail (nunits units of U quads); warp-uniform trip count: every
        // lane iterates until the warp's first quad is past the end (lanes past it hash nothing)
        const uint32_t nq = nunits * U;
        for (uint32_t ub = u - lane; ub < nq; ub += stride) {
            const uint32_t uu = ub + lane;
            if (Sh::ANY_HLL && it == next_refresh) {
                next_refresh = it + min(it, 32u);
#pragma unroll
                for (int s = 0; s < NC; ++s)
                    if (Sh::active(P, s) && Sh::hll(P, s) && !Sh::hllbm(P, s) && !((bmfull >> s) & 1u)) {
                        const uint32_t hc = P.slot[s].hceil_off;
                        const uint32_t hb = hll_bound(Sh::hllw(P, s), P.g_hll_glob + Sh::hllout(P, s) * kHllM, s,
                                                      hc != kNone ? P.g_hceil + hc : nullptr);
                        const uint32_t L = min(hb & 255u, 31u);
                        if (lane == 0) wlim[s] = (0xFFFFFFFFu >> L) & 0xFFFFFFFEu;
                        if (hb >> 8) bmfull |= 1u << s;
                    } else if (Sh::active(P, s) && Sh::hll(P, s) && Sh::hllbm(P, s) && !((bmfull >> s) & 1u) &&
                               P.slot[s].bm_words <= kBmRefreshWords &&
                               bm_push(smem32() + Sh::bmaddr(P, s) / 4, P.g_bm + P.slot[s].bm_goff,
                                       P.slot[s].bm_words, P.g_bmcnt + s, Sh::bmnv(P, s)))
                        bmfull |= 1u << s;
                __syncwarp();
            }
            ++it;
            // hashed past the end too (pure arithmetic), masked: no branch around the hash
            const uint32_t keep = quad_keep(uu) & (uu < nq ? 0xFu : 0u);
            const uint32_t c = __popc(keep);
            kept += c;
            if (!__ballot_sync(0xFFFFFFFFu, keep)) continue;      // no kept row in the warp's 128
            // one warp prefix sum of the lanes' kept-row counts places every kept row of the
            // iteration at once (instead of a ballot per quad row)
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            if (qt - qh + total <= kQueue) {
                uint32_t pos = qt + incl - c, m = keep;
                while (m) {
                    q[pos++ % kQueue] = uu * 4 + (__ffs(m) - 1);
                    m &= m - 1;
                }
                qt += total;
                __syncwarp();
                while (qt - qh >= 32) work(32);
            } else {                                   // > 64 - pending at once: row by row
#pragma unroll
                for (int k = 0; k < 4; ++k) {          // row k of every lane's quad: <= 32 new entries
                    const uint32_t b = __ballot_sync(0xFFFFFFFFu, (keep >> k) & 1u);
                    if (!b) continue;
                    if ((b >> lane) & 1u) q[(qt + __popc(b & ((1u << lane) - 1u))) % kQueue] = uu * 4 + k;
                    qt += __popc(b);
                    __syncwarp();
                    if (qt - qh >= 32) work(32);
                }
            }
        }
        if (qt != qh) work(qt - qh);                  // the last partial batch
    } else if (U == 1 && NC <= 4) {
        // column-streamed loop; a sampled probe loads only quads with a kept row (at rate
        // 0.01 that is 4 % of the quads, so most key bytes are never read)
        int4 r[NC][Sh::I64 ? 2 : 1];
        uint32_t keep = u < nunits ? quad_keep(u) : 0u;
        if (keep) {
#pragma unroll
            for (int s = 0; s < NC; ++s)
                if (Sh::active(P, s)) load_col<Sh>(P, s, u, r[s]);
        }
        for (; u < nunits; u += stride) {
#if GACE_L2_PREFETCH
            // keys two iterations ahead pulled into L2, so the register loads of the next
            // iteration hit L2 (full scans only: a sampled probe must not fetch the rows it skips).
            // GACE_L2_PREFETCH=2 (int32 columns): one 128-byte line per lane -- lane l takes line
            // l % 4 of column l / 4 (the warp's 512 bytes of a column are 4 lines), so a single
            // PREFETCH covers every column.  (cp.async.bulk.prefetch needs a warp-uniform
            // address: the compiler wraps it in a per-lane loop.)  Otherwise one PREFETCH per
            // column, each lane its own 16 (32) bytes.
            if (GACE_L2_PREFETCH == 3 && !Sh::I64) {
                // int32 plans: no prefetch (the column-streamed register loads keep enough
                // bytes in flight)
            } else if (GACE_L2_PREFETCH == 2 && !Sh::I64 && NC <= 8) {
                if (!Sh::SAMPLE) {
                    const uint32_t lane = threadIdx.x & 31u;
                    const uint32_t upf = u - lane + GACE_L2_PF_DIST * stride + 8u * (lane & 3u);
                    const int s = (int)(lane >> 2);
                    if (s < NC && upf < nunits && Sh::active(P, s))
                        asm volatile("prefetch.global.L2 [%0];" ::
                                     "l"(static_cast<const char *>(P.slot[s].ptr) + (uint64_t)upf * 16u));
                }
            } else if (!Sh::SAMPLE && u + GACE_L2_PF_DIST * stride < nunits) {
#pragma unroll
                for (int s = 0; s < NC; ++s) {
                    if (!Sh::active(P, s)) continue;
                    const uint32_t w = Sh::is32(P, s) ? 16u : 32u;
                    const char *a = static_cast<const char *>(P.slot[s].ptr) + (uint64_t)(u + GACE_L2_PF_DIST * stride) * w;
                    asm volatile("prefetch.global.L2 [%0];" :: "l"(a));
                    if (w == 32u) asm volatile("prefetch.global.L2 [%0];" :: "l"(a + 16));
                }
            }
#endif
            uint32_t un = u + stride < nunits ? u + stride : kNoUnit;
            const uint32_t keep_n = un != kNoUnit ? quad_keep(un) : 0u;
            if (!keep_n) un = kNoUnit;
            if (Sh::ANY_HLL && it == next_refresh) {
                next_refresh = it + min(it, 32u);
                if (__activemask() == 0xFFFFFFFFu) {
#pragma unroll
                    for (int s = 0; s < NC; ++s)
                        if (Sh::active(P, s) && Sh::hll(P, s) && !Sh::hllbm(P, s) && !((bmfull >> s) & 1u)) {
                            const uint32_t hc = P.slot[s].hceil_off;
                            const uint32_t hb = hll_bound(Sh::hllw(P, s), P.g_hll_glob + Sh::hllout(P, s) * kHllM, s,
                                                          hc != kNone ? P.g_hceil + hc : nullptr);
                            const uint32_t L = min(hb & 255u, 31u);
                            if ((threadIdx.x & 31) == 0) wlim[s] = (0xFFFFFFFFu >> L) & 0xFFFFFFFEu;
                            if (hb >> 8) bmfull |= 1u << s;       // registers at their ceilings: column complete
                        }
                        else if (Sh::active(P, s) && Sh::hll(P, s) && Sh::hllbm(P, s) && !((bmfull >> s) & 1u) &&
                                 P.slot[s].bm_words <= kBmRefreshWords &&
                                 bm_push(smem32() + Sh::bmaddr(P, s) / 4, P.g_bm + P.slot[s].bm_goff,
                                         P.slot[s].bm_words, P.g_bmcnt + s, Sh::bmnv(P, s)))
                            bmfull |= 1u << s;
                    __syncwarp();
                }
            }
            ++it;
            if (Sh::SAMPLE) kept += __popc(keep);
            if (keep) {
                quad_work<Sh>(P, r, keep, wlim, bmfull, un);
            } else if (un != kNoUnit) {        // nothing kept here: start the next unit's loads
#pragma unroll
                for (int s = 0; s < NC; ++s)
                    if (Sh::active(P, s)) load_col<Sh>(P, s, un, r[s]);
            }
            keep = keep_n;
        }
    } else {
#if GACE_PREFETCH
    Unit<Sh> X;
    if (u < nunits) load_unit<Sh>(P, u, X);
    for (; u < nunits; u += stride) {
        Unit<Sh> Xn;
        if (u + stride < nunits) load_unit<Sh>(P, u + stride, Xn);       // prefetch
        body(X, u);
        X = Xn;
    }
#else
    // no register prefetch: the 32 warps of the SM keep loads in flight, and the registers go
    // to the lookup / hash work instead; the units two iterations ahead are pulled into L2
    for (; u < nunits; u += stride) {
#if GACE_L2_PREFETCH_U
        if (!Sh::SAMPLE && u + 2 * stride < nunits) {
#pragma unroll
            for (int s = 0; s < NC; ++s) {
                if (!Sh::active(P, s)) continue;
                const char *a = static_cast<const char *>(P.slot[s].ptr) +
                                (uint64_t)(u + 2 * stride) * U * (Sh::is32(P, s) ? 16u : 32u);
                asm volatile("prefetch.global.L2 [%0];" :: "l"(a));
            }
        }
#endif
        Unit<Sh> X;
        load_unit<Sh>(P, u, X);
        body(X, u);
    }
#endif
    }
    if (!Sh::SAMPLE) kept += 4 * U * it;   // every row of every unit this thread processed
    // tail rows [nunits * 4U, nrows): one row per thread of the last CTA
    const uint64_t tail0 = (uint64_t)nunits * (4 * U);   // 64-bit: a launch may hold 2^33 rows
    if (blockIdx.x == gridDim.x - 1 && tail0 + threadIdx.x < P.nrows) kept += tail_row<Sh>(P, tail0 + threadIdx.x);
    __syncthreads();

    // CTA partials -> global
    for (uint32_t i = threadIdx.x; i < P.acc_words; i += blockDim.x) {
        const uint32_t x = sm[P.acc_idx + i];
        if (x) atomicAdd(P.g_acc + i, (unsigned long long)x);
    }
#pragma unroll 1
    for (int s = 0; s < NC; ++s) {
        if (!Sh::active(P, s) || !Sh::hll(P, s)) continue;
        if (Sh::hllbm(P, s)) {           // presence bitmap -> OR into the merged bitmap
            const uint32_t *src = smem32() + Sh::bmaddr(P, s) / 4;
            uint32_t *dst = P.g_bm + P.slot[s].bm_goff;
            for (uint32_t i = threadIdx.x; i < P.slot[s].bm_words; i += blockDim.x)
                if (src[i]) atomicOr(dst + i, src[i]);
            continue;
        }
        // u32 registers -> packed u8 partial of this CTA (its output block; a bitmap
        // column's block stays zero and is filled by fin_bitmap_hll)
        const uint4 *src = reinterpret_cast<const uint4 *>(smem32() + Sh::hllw(P, s));
        uint32_t *dst = reinterpret_cast<uint32_t *>(P.g_hll_part + (size_t)blockIdx.x * P.hll_bytes +
                                                     (size_t)Sh::hllout(P, s) * kHllM);
        for (uint32_t i = threadIdx.x; i < kHllM / 4; i += blockDim.x) {
            const uint4 q = src[i];
            uint32_t x = q.x | (q.y << 8) | (q.z << 16) | (q.w << 24);
            if (P.part_merge) x = __vmaxu4(x, dst[i]);   // later launch of a chunked probe
            dst[i] = x;
        }
    }
    if (P.hll_bytes && !P.part_merge) {  // bitmap columns' blocks of the partial: zeros
#pragma unroll 1
        for (int s = 0; s < NC; ++s) {
            if (!Sh::active(P, s) || !Sh::hll(P, s) || !Sh::hllbm(P, s)) continue;
            uint32_t *dst = reinterpret_cast<uint32_t *>(P.g_hll_part + (size_t)blockIdx.x * P.hll_bytes +
                                                         (size_t)Sh::hllout(P, s) * kHllM);
            for (uint32_t i = threadIdx.x; i < kHllM / 4; i += blockDim.x) dst[i] = 0u;
        }
    }
    kept = __reduce_add_sync(0xFFFFFFFFu, kept);
    if ((threadIdx.x & 31) == 0 && kept) atomicAdd(P.g_nsamp, (unsigned long long)kept);
}

}  // namespace gace
