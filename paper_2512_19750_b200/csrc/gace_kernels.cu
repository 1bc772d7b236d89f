// gace_kernels.cu -- sm_100a kernels of the GACE selectivity probe.
//
// Hot path: probe_kernel streams every probed key
// column once from HBM with 128-bit non-allocating loads, draws the Bernoulli
// sample bit from a counter-based SplitMix64 of the global row id, resolves each
// value's bucket with a shared-memory lookup table, and accumulates
//   * a per-column u32 bucket histogram   (-> counts by prefix differences),
//   * a per-column-pair 2-D sub-bucket grid (-> joint counts by rectangle sums),
//   * u8 HyperLogLog registers            (fmix32 / mix64 hash, read-check-CAS max),
// all in shared memory.  One CTA per SM, grid-stride over row quads.  At the
// end each CTA adds its nonzero bins into global u64 accumulators and writes
// its HLL registers as a per-CTA partial.  fin_prefix / fin_output turn the
// accumulators into the packed result [n_sampled, counts, joints] + registers.
// No tensor cores: this is an HBM-bound integer scan.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "gace_kernels.h"
#include "gace_plan.h"

namespace gace {

#define GACE_GAMMA 0x9E3779B97F4A7C15ULL

// SplitMix64 finaliser (sample bit; int64 HLL hash).  DESIGN.md "Semantics" 1, 6.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// MurmurHash3 fmix32 (int32 HLL hash).  DESIGN.md "Semantics" 6.
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

// HLL registers live in shared memory as u32 (native ATOMS.MAX; registers only grow).
// `lmin` is a lower bound on every register of the column in this CTA (refreshed now
// and then); a value with rank <= lmin cannot raise any register and skips the
// shared-memory check entirely -- after warm-up that is nearly every value.
__device__ __forceinline__ void hll_update(const SlotParams &S, uint32_t idx, uint32_t r, uint32_t lmin,
                                           uint32_t dbg) {
    if (r <= lmin) return;
    uint32_t *R = reinterpret_cast<uint32_t *>(g_smem) + S.hll_idx;
    if (r > R[idx] && !(dbg & 1)) atomicMax(R + idx, r);
}

__device__ __forceinline__ void hll_i32(const SlotParams &S, int32_t x, uint32_t lmin, uint32_t dbg) {
    const uint32_t h = fmix32(static_cast<uint32_t>(x));
    const uint32_t r = __clz((h << kHllP) | (1u << (kHllP - 1))) + 1;   // <= 32-p+1
    hll_update(S, h >> (32 - kHllP), r, lmin, dbg);
}

__device__ __forceinline__ void hll_i64(const SlotParams &S, int64_t x, uint32_t lmin, uint32_t dbg) {
    const uint64_t h = mix64(static_cast<uint64_t>(x) + GACE_GAMMA);
    const uint32_t r = __clzll((h << kHllP) | (1ull << (kHllP - 1))) + 1;  // <= 64-p+1
    hll_update(S, static_cast<uint32_t>(h >> (64 - kHllP)), r, lmin, dbg);
}

// Warp-cooperative exact minimum of a column's 4096 registers (whole warp active).
__device__ __noinline__ uint32_t hll_min(const SlotParams &S) {
    const uint4 *R = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint32_t *>(g_smem) + S.hll_idx);
    const uint32_t lane = threadIdx.x & 31;
    uint32_t m = 0xFFFFFFFFu;
#pragma unroll 8
    for (int i = 0; i < kHllM / 4 / 32; ++i) {
        const uint4 v = R[i * 32 + lane];
        m = min(m, min(min(v.x, v.y), min(v.z, v.w)));
    }
    return __reduce_min_sync(0xFFFFFFFFu, m);
}

// #{t in bps : t <= v}, branch-free binary search (MODE_SEARCH fallback; kept out of line
// so the hot loop stays small enough for the instruction cache).
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
    __device__ __forceinline__ uint2 u2(uint32_t i) const { return reinterpret_cast<const uint2 *>(g_smem)[i]; }
    __device__ __forceinline__ uint32_t u32(uint32_t i) const { return reinterpret_cast<const uint32_t *>(g_smem)[i]; }
};

// Absolute shared-memory index of the histogram bucket of offset u (full walk through
// nested cells and lists; out of line, only taken for the rare special entries).
__device__ __noinline__ uint32_t lut_bucket(const SlotParams &S, uint32_t u) {
    return lut_lookup(SmemTables{}, S.lut_idx, S.s1, u);
}

__device__ __forceinline__ uint32_t bucket_i32(const SlotParams &S, int32_t x, bool clamp) {
    if (S.mode == MODE_SEARCH) return S.hist_idx + search_bucket(S.bps, S.nbp, x);
    if (clamp) x = min(max(x, static_cast<int32_t>(S.clamp_lo)), static_cast<int32_t>(S.clamp_hi));
    return lut_bucket(S, static_cast<uint32_t>(x) - static_cast<uint32_t>(S.base));
}

__device__ __forceinline__ uint32_t bucket_i64(const SlotParams &S, int64_t x, bool clamp) {
    if (S.mode == MODE_SEARCH) return S.hist_idx + search_bucket(S.bps, S.nbp, x);
    if (clamp) x = min(max(x, S.clamp_lo), S.clamp_hi);
    return lut_bucket(S, static_cast<uint32_t>(static_cast<uint64_t>(x) - static_cast<uint64_t>(S.base)));
}

__device__ __forceinline__ bool keep_row(const ProbeParams &P, uint64_t g) {
    return mix64(P.seed + (g + 1) * GACE_GAMMA) < P.thr;
}

// Register-resident 16-byte chunks of one "unit" (U row quads) of every slot: the
// main loop prefetches the next unit's chunks while it processes this one.
template <int NC, int U, bool I64>
struct Unit {
    int4 r[NC][U][I64 ? 2 : 1];
};

template <int NC, int U, bool I64>
__device__ __forceinline__ void load_unit(const ProbeParams &P, uint64_t u, Unit<NC, U, I64> &X) {
#pragma unroll
    for (int s = 0; s < NC; ++s) {
        if (s >= (int)P.nslots) continue;
        const char *base = static_cast<const char *>(P.slot[s].ptr);
        if (!I64 || P.slot[s].dtype == 0) {
#pragma unroll
            for (int j = 0; j < U; ++j) X.r[s][j][0] = ld_stream(base + (u * U + j) * 16);
        } else {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                X.r[s][j][0] = ld_stream(base + (u * U + j) * 32);
                X.r[s][j][I64 ? 1 : 0] = ld_stream(base + (u * U + j) * 32 + 16);
            }
        }
    }
}

// Keys of one slot's row quad: int64 only in kernels that have an int64 column.
template <bool I64>
using KeyT = typename std::conditional<I64, int64_t, int32_t>::type;

template <bool I64>
__device__ __forceinline__ void decode(const SlotParams &S, const int4 (&r)[I64 ? 2 : 1], KeyT<I64> (&v)[4]) {
    if (!I64 || S.dtype == 0) {
        v[0] = r[0].x; v[1] = r[0].y; v[2] = r[0].z; v[3] = r[0].w;
    } else {
        v[0] = static_cast<KeyT<I64>>((static_cast<int64_t>(r[0].y) << 32) | static_cast<uint32_t>(r[0].x));
        v[1] = static_cast<KeyT<I64>>((static_cast<int64_t>(r[0].w) << 32) | static_cast<uint32_t>(r[0].z));
        v[2] = static_cast<KeyT<I64>>((static_cast<int64_t>(r[I64 ? 1 : 0].y) << 32) | static_cast<uint32_t>(r[I64 ? 1 : 0].x));
        v[3] = static_cast<KeyT<I64>>((static_cast<int64_t>(r[I64 ? 1 : 0].w) << 32) | static_cast<uint32_t>(r[I64 ? 1 : 0].z));
    }
}

// Offset u = key - base of a LUT-mode slot (with the optional clamp), 32-bit ops for int32.
template <bool I64>
__device__ __forceinline__ uint32_t offset_of(const SlotParams &S, KeyT<I64> xk, bool clamp) {
    if (!I64 || S.dtype == 0) {
        int32_t y = static_cast<int32_t>(xk);
        if (clamp) y = min(max(y, static_cast<int32_t>(S.clamp_lo)), static_cast<int32_t>(S.clamp_hi));
        return static_cast<uint32_t>(y) - static_cast<uint32_t>(S.base);
    }
    int64_t x = xk;
    if (clamp) x = min(max(x, S.clamp_lo), S.clamp_hi);
    return static_cast<uint32_t>(static_cast<uint64_t>(x) - static_cast<uint64_t>(S.base));
}

// Absolute bucket ids of a row quad, 16 bits per slot (shared-memory u32 index < 2^16),
// four slots per 64-bit word: extraction by a runtime slot index is a shift, so the
// pair loop below can run over groups without spilling a per-slot array.
template <int NC>
struct Ids {
    uint64_t w[(NC + 3) / 4][4];
    __device__ __forceinline__ void set(int s, int k, uint32_t b) {   // s compile-time
        w[s >> 2][k] |= static_cast<uint64_t>(b) << (16 * (s & 3));
    }
    __device__ __forceinline__ uint32_t get(uint32_t s, int k) const {
        const uint64_t x = (NC > 4 && (s & 4)) ? w[(NC + 3) / 4 - 1][k] : w[0][k];
        return static_cast<uint32_t>(x >> (16 * (s & 3))) & 0xFFFFu;
    }
};

// Buckets of slots [S0, S0 + NB) over one row quad.  All level-1 lookups are issued
// before any is consumed; the rare nested / list / search entries are resolved
// afterwards behind one branch.
template <int NC, int S0, int NB, bool I64>
__device__ __forceinline__ void buckets_batch(const ProbeParams &P, const KeyT<I64> (&v)[NC][4], Ids<NC> &ids) {
    const uint2 *T = reinterpret_cast<const uint2 *>(g_smem);
    const bool clamp = P.clamp;
    uint32_t u[NB][4];
    uint2 e[NB][4];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const SlotParams &S = P.slot[S0 + i];
        const bool lut = S0 + i < (int)P.nslots && S.mode == MODE_LUT;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            u[i][k] = lut ? offset_of<I64>(S, v[S0 + i][k], clamp) : 0u;
            e[i][k] = lut ? T[S.lut_idx + (u[i][k] >> S.s1)] : make_uint2(0u, 0u);
        }
    }
    uint32_t spec = 0;
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) spec |= e[i][k].x;
    if (spec & kSpecial) {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const SlotParams &S = P.slot[S0 + i];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (e[i][k].x & kSpecial) e[i][k] = make_uint2(lut_bucket(S, u[i][k]), kNoThr);
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int s = S0 + i;
        const SlotParams &S = P.slot[s];
        if (s < (int)P.nslots && S.mode == MODE_SEARCH) {      // binary-search fallback column
#pragma unroll
            for (int k = 0; k < 4; ++k) e[i][k] = make_uint2(S.hist_idx + search_bucket(S.bps, S.nbp, v[s][k]), kNoThr);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) ids.set(s, k, (e[i][k].x & kBaseMask) + (u[i][k] > e[i][k].y ? 1u : 0u));
    }
}

// Rows per thread per loop iteration: 4 * U, U chosen so each thread keeps >= 64 bytes
// of every column in flight (plus the same again prefetched).
template <int NC>
struct Cfg {
    static constexpr int U = NC >= 4 ? 1 : 4 / NC;
};

// Everything one row quad contributes: histograms, HLL registers, 2-D pair grids and
// per-row ("direct") pairs.  keep: one bit per row.
template <int NC, bool I64>
__device__ __forceinline__ void quad_work(const ProbeParams &P, const int4 (&r)[NC][I64 ? 2 : 1], uint32_t keep,
                                          const uint32_t (&lmin)[NC]) {
    uint32_t *sm32 = reinterpret_cast<uint32_t *>(g_smem);
    const uint32_t dbg = P.dbg;
    KeyT<I64> v[NC][4];
#pragma unroll
    for (int s = 0; s < NC; ++s)
        if (s < (int)P.nslots) decode<I64>(P.slot[s], r[s], v[s]);
    Ids<NC> ids;
#pragma unroll
    for (int h = 0; h < (NC + 3) / 4; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) ids.w[h][k] = 0;
    buckets_batch<NC, 0, (NC < 4 ? NC : 4), I64>(P, v, ids);
    if (NC > 4) buckets_batch<NC, (NC > 4 ? 4 : 0), (NC > 4 ? NC - 4 : 1), I64>(P, v, ids);
    // per-column bucket histograms
#pragma unroll
    for (int s = 0; s < NC; ++s) {
        if (s >= (int)P.nslots || P.slot[s].mode == MODE_NOPRED || (dbg & 2)) continue;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((keep >> k) & 1u) atomicAdd(sm32 + ids.get(s, k), 1u);
    }
    // HLL: hash all four keys, then one branch for the (rare) ranks above the bound
#pragma unroll
    for (int s = 0; s < NC; ++s) {
        const SlotParams &S = P.slot[s];
        if (s >= (int)P.nslots || !S.has_hll || (dbg & 8)) continue;
        uint32_t idx[4], rk[4], m = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!I64 || S.dtype == 0) {
                const uint32_t h = fmix32(static_cast<uint32_t>(v[s][k]));
                idx[k] = h >> (32 - kHllP);
                rk[k] = __clz((h << kHllP) | (1u << (kHllP - 1))) + 1;
            } else {
                const uint64_t h = mix64(static_cast<uint64_t>(v[s][k]) + GACE_GAMMA);
                idx[k] = static_cast<uint32_t>(h >> (64 - kHllP));
                rk[k] = __clzll((h << kHllP) | (1ull << (kHllP - 1))) + 1;
            }
            // a key equal to the previous kept row's key cannot change a register
            const bool dup = k > 0 && ((keep >> (k - 1)) & 1u) && v[s][k] == v[s][k - 1];
            m |= (((keep >> k) & 1u) && !dup && rk[k] > lmin[s]) ? (1u << k) : 0u;
        }
        if (m) {
            uint32_t *R = sm32 + S.hll_idx;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (((m >> k) & 1u) && rk[k] > R[idx[k]] && !(dbg & 1)) atomicMax(R + idx[k], rk[k]);
        }
    }
    // pairs: runtime loop over column pairs
    for (uint32_t g = 0; g < P.ngroups; ++g) {
        const GroupParams &G = P.grp[g];
        if (G.has_grid && !(dbg & 4)) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if ((keep >> k) & 1u) {
                    const uint32_t ia = sm32[G.mapA_adj + (int)ids.get(G.a, k)];
                    const uint32_t ib = sm32[G.mapB_adj + (int)ids.get(G.b, k)];
                    atomicAdd(sm32 + ia + ib, 1u);
                }
            }
        }
        for (uint32_t d = G.dbeg; d < G.dend; ++d) {
            const DirectPair D = P.direct[d];
            uint32_t c = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t ba = ids.get(G.a, k), bb = ids.get(G.b, k);
                const uint32_t ina = ((ba >= D.la) & (ba <= D.ha)) ^ D.nega;
                const uint32_t inb = ((bb >= D.lb) & (bb <= D.hb)) ^ D.negb;
                c += ((keep >> k) & 1u) & ina & inb;
            }
            // per-thread add: this loop may run with a diverged warp (sampled quads), where a
            // warp-collective reduction over __activemask() is not well defined
            if (c) atomicAdd(sm32 + D.acc_idx, c);
        }
    }
}

// One row past the last full unit (scalar loads; out of line: cold code).
template <int NC, bool SAMPLE, bool I64>
__device__ __noinline__ uint32_t tail_row(const ProbeParams &P, uint64_t r) {
    const uint32_t keep = (!SAMPLE || keep_row(P, P.row0 + r)) ? 1u : 0u;
    if (!keep) return 0;
    int4 rj[NC][I64 ? 2 : 1];
#pragma unroll
    for (int s = 0; s < NC; ++s) {
        if (s >= (int)P.nslots) continue;
        if (!I64 || P.slot[s].dtype == 0) {
            const int32_t x = __ldg(static_cast<const int32_t *>(P.slot[s].ptr) + r);
            rj[s][0] = make_int4(x, x, x, x);     // rows 1..3 of the quad are masked off
        } else {
            const long long x = __ldg(static_cast<const long long *>(P.slot[s].ptr) + r);
            const int lo = (int)(x & 0xFFFFFFFF), hi = (int)(x >> 32);
            rj[s][0] = make_int4(lo, hi, lo, hi);
            rj[s][I64 ? 1 : 0] = make_int4(lo, hi, lo, hi);
        }
    }
    uint32_t zero[NC];
#pragma unroll
    for (int s = 0; s < NC; ++s) zero[s] = 0;
    quad_work<NC, I64>(P, rj, 1u, zero);
    return 1;
}

template <int NC, bool SAMPLE, bool I64>
__global__ void __launch_bounds__(kThreads, 1) probe_kernel(const __grid_constant__ ProbeParams P) {
    constexpr int U = Cfg<NC>::U;
    uint32_t *sm32 = reinterpret_cast<uint32_t *>(g_smem);
    // tables -> shared memory; accumulators and registers -> 0
    for (uint32_t i = threadIdx.x; i < P.image_u4; i += blockDim.x) g_smem[i] = __ldg(P.image + i);
    for (uint32_t i = P.image_u4 + threadIdx.x; i < P.smem_bytes / 16; i += blockDim.x)
        g_smem[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();

    const uint64_t nunits = P.nrows / (4 * U);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t kept = 0;
    uint32_t lmin[NC];
#pragma unroll
    for (int s = 0; s < NC; ++s) lmin[s] = 0;
    uint32_t it = 0, next_refresh = 4;
    uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    Unit<NC, U, I64> X;
    if (u < nunits) load_unit(P, u, X);
    for (; u < nunits; u += stride, ++it) {
        Unit<NC, U, I64> Xn;
        if (u + stride < nunits) load_unit(P, u + stride, Xn);           // prefetch
        if (it == next_refresh) {
            next_refresh = it + min(it, 128u);
            if (__activemask() == 0xFFFFFFFFu) {
#pragma unroll
                for (int s = 0; s < NC; ++s)
                    if (s < (int)P.nslots && P.slot[s].has_hll) lmin[s] = hll_min(P.slot[s]);
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            uint32_t keep = 0xFu;
            if (SAMPLE) {
                const uint64_t g0 = P.row0 + (u * U + j) * 4;
                keep = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) keep |= (keep_row(P, g0 + k) ? 1u : 0u) << k;
                kept += __popc(keep);
                if (!keep) continue;
            }
            int4 rj[NC][I64 ? 2 : 1];
#pragma unroll
            for (int s = 0; s < NC; ++s) {
                rj[s][0] = X.r[s][j][0];
                if (I64) rj[s][I64 ? 1 : 0] = X.r[s][j][I64 ? 1 : 0];
            }
            quad_work<NC, I64>(P, rj, keep, lmin);
        }
        X = Xn;
    }
    if (!SAMPLE) kept += 4 * U * it;   // every row of every unit this thread processed was kept
    // tail rows [nunits * 4U, nrows): one row per thread of the last CTA, scalar loads
    const uint64_t tail0 = nunits * 4 * U;
    if (blockIdx.x == gridDim.x - 1 && tail0 + threadIdx.x < P.nrows)
        kept += tail_row<NC, SAMPLE, I64>(P, tail0 + threadIdx.x);
    __syncthreads();

    // CTA partials -> global
    for (uint32_t i = threadIdx.x; i < P.acc_words; i += blockDim.x) {
        const uint32_t v = sm32[P.acc_idx + i];
        if (v) atomicAdd(P.g_acc + i, (unsigned long long)v);
    }
    if (P.hll_bytes) {   // u32 registers -> packed u8 partial of this CTA
        const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint8_t *>(g_smem) + P.hll_off);
        uint32_t *dst = reinterpret_cast<uint32_t *>(P.g_hll_part + (size_t)blockIdx.x * P.hll_bytes);
        for (uint32_t i = threadIdx.x; i < P.hll_bytes / 4; i += blockDim.x) {
            const uint4 r = src[i];
            uint32_t v = r.x | (r.y << 8) | (r.z << 16) | (r.w << 24);
            if (P.part_merge) v = __vmaxu4(v, dst[i]);   // later launch of a chunked probe
            dst[i] = v;
        }
    }
    kept = __reduce_add_sync(0xFFFFFFFFu, kept);
    if ((threadIdx.x & 31) == 0 && kept) atomicAdd(P.g_nsamp, (unsigned long long)kept);
}

// ------------------------------------------------------------------ finalize

__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                   unsigned long long *total) {
    __shared__ unsigned long long warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) / 32;
        unsigned long long s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) warp_sums[lane] = s;     // inclusive
    }
    __syncthreads();
    const unsigned long long before = (wid ? warp_sums[wid - 1] : 0) + x - v;
    *total = warp_sums[(blockDim.x + 31) / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(1024) fin_prefix(const FinParams F) {
    if (blockIdx.x < F.njobs) {
        const FinJob J = F.jobs[blockIdx.x];
        const unsigned long long *src = F.g_acc + J.src;
        unsigned long long *dst = F.g_pre + J.dst;
        if (J.kind == JOB_HIST) {
            const uint32_t n = J.nb;
            const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
            const uint32_t beg = min(n, threadIdx.x * per), end = min(n, beg + per);
            unsigned long long s = 0;
            for (uint32_t i = beg; i < end; ++i) s += src[i];
            unsigned long long total;
            unsigned long long run = block_exclusive_scan(s, &total);
            for (uint32_t i = beg; i < end; ++i) {
                dst[i] = run;
                run += src[i];
            }
            if (threadIdx.x == 0) dst[n] = total;
        } else {   // JOB_SAT: summed-area table with a zero border, row stride nb + 1
            const uint32_t na = J.na, nb = J.nb, st = nb + 1;
            for (uint32_t j = threadIdx.x; j <= nb; j += blockDim.x) dst[j] = 0;
            for (uint32_t i = threadIdx.x; i < na; i += blockDim.x) {
                unsigned long long run = 0;
                dst[(size_t)(i + 1) * st] = 0;
                for (uint32_t j = 0; j < nb; ++j) {
                    run += src[(size_t)i * nb + j];
                    dst[(size_t)(i + 1) * st + j + 1] = run;
                }
            }
            __syncthreads();
            for (uint32_t j = threadIdx.x; j < nb; j += blockDim.x) {
                unsigned long long run = 0;
                for (uint32_t i = 0; i < na; ++i) {
                    run += dst[(size_t)(i + 1) * st + j + 1];
                    dst[(size_t)(i + 1) * st + j + 1] = run;
                }
            }
        }
    } else {   // HLL: byte-wise max over the per-CTA partials
        const uint32_t words = F.hll_bytes / 4;
        const uint32_t b = blockIdx.x - F.njobs;
        const uint32_t per = (words + F.hll_blocks - 1) / F.hll_blocks;
        const uint32_t beg = b * per, end = min(words, beg + per);
        const uint32_t *part = reinterpret_cast<const uint32_t *>(F.g_hll_part);
        for (uint32_t w = beg + threadIdx.x; w < end; w += blockDim.x) {
            uint32_t m = 0;
            for (uint32_t c = 0; c < F.nparts; ++c) m = __vmaxu4(m, part[(size_t)c * words + w]);
            reinterpret_cast<uint32_t *>(F.out_regs)[w] = m;
        }
    }
}

__device__ __forceinline__ unsigned long long iv(const unsigned long long *pre, uint32_t lo, uint32_t hi) {
    return lo <= hi ? pre[hi + 1] - pre[lo] : 0ull;
}

__device__ __forceinline__ unsigned long long rect(const unsigned long long *S, uint32_t st, uint32_t r0,
                                                   uint32_t r1, uint32_t c0, uint32_t c1) {
    if (r0 > r1 || c0 > c1) return 0ull;
    return S[(size_t)(r1 + 1) * st + c1 + 1] - S[(size_t)r0 * st + c1 + 1] - S[(size_t)(r1 + 1) * st + c0] +
           S[(size_t)r0 * st + c0];
}

// joint of (p_i xor neg_i) and (p_j xor neg_j) from c_i = |p_i|, c_j = |p_j|, c_ij = |p_i and p_j|
__device__ __forceinline__ unsigned long long combine(unsigned long long n, unsigned long long ci,
                                                      unsigned long long cj, unsigned long long cij,
                                                      uint32_t ni, uint32_t nj) {
    if (!ni && !nj) return cij;
    if (ni && !nj) return cj - cij;
    if (!ni && nj) return ci - cij;
    return n - ci - cj + cij;
}

__global__ void fin_output(const FinParams F) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long n = *F.g_nsamp;
    if (t == 0) F.out[0] = n;
    if (t >= 1 && t <= F.npreds) {
        const FinPred p = F.preds[t - 1];
        const unsigned long long c = iv(F.g_pre + p.pre, p.lo, p.hi);
        F.out[t] = p.neg ? n - c : c;
    } else if (t > F.npreds && t <= F.npreds + F.npairs) {
        const FinPair q = F.pairs[t - 1 - F.npreds];
        unsigned long long r;
        if (q.kind == PAIR_DIRECT) {
            r = F.g_acc[q.pre];
        } else if (q.kind == PAIR_SAME) {
            const unsigned long long *pre = F.g_pre + q.pre;
            const uint32_t lo = max(q.li, q.lj), hi = min(q.hi, q.hj);
            r = combine(n, iv(pre, q.li, q.hi), iv(pre, q.lj, q.hj), iv(pre, lo, hi), q.negi, q.negj);
        } else {
            const unsigned long long *S = F.g_pre + q.pre;
            const uint32_t st = q.nb + 1;
            const unsigned long long ci = rect(S, st, q.li, q.hi, 0, q.nb - 1);
            const unsigned long long cj = rect(S, st, 0, q.na - 1, q.lj, q.hj);
            const unsigned long long cij = rect(S, st, q.li, q.hi, q.lj, q.hj);
            r = combine(n, ci, cj, cij, q.negi, q.negj);
        }
        F.out[t] = r;
    }
}

// ------------------------------------------------------------------ attach / test hook

__global__ void minmax_kernel(const void *col, int dtype, uint64_t n, long long *mm) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long v = dtype == 0 ? (long long)__ldg(static_cast<const int32_t *>(col) + i)
                                       : __ldg(static_cast<const long long *>(col) + i);
        lo = min(lo, v);
        hi = max(hi, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

__global__ void sample_mask_kernel(uint64_t nrows, uint64_t row0, uint64_t seed, uint64_t thr,
                                   uint32_t all, unsigned long long *bits) {
    const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w * 64 >= nrows) return;
    unsigned long long m = 0;
    for (int b = 0; b < 64; ++b) {
        const uint64_t r = w * 64 + b;
        if (r >= nrows) break;
        const uint64_t g = row0 + r;
        if (all || mix64(seed + (g + 1) * GACE_GAMMA) < thr) m |= 1ull << b;
    }
    bits[w] = m;
}

// ------------------------------------------------------------------ launchers

template <int NC, bool SAMPLE, bool I64>
static cudaError_t launch_t(const ProbeParams &P, int grid, cudaStream_t s) {
    auto k = probe_kernel<NC, SAMPLE, I64>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    k<<<grid, kThreads, P.smem_bytes, s>>>(P);
    return cudaGetLastError();
}

template <int NC>
static cudaError_t launch_nc(const ProbeParams &P, bool sample, bool i64, int grid, cudaStream_t s) {
    if (i64) return sample ? launch_t<NC, true, true>(P, grid, s) : launch_t<NC, false, true>(P, grid, s);
    return sample ? launch_t<NC, true, false>(P, grid, s) : launch_t<NC, false, false>(P, grid, s);
}

cudaError_t launch_probe(const ProbeParams &P, bool sample, bool i64, int grid, cudaStream_t s) {
    const uint32_t n = P.nslots;
    if (n <= 1) return launch_nc<1>(P, sample, i64, grid, s);
    if (n <= 2) return launch_nc<2>(P, sample, i64, grid, s);
    if (n <= 4) return launch_nc<4>(P, sample, i64, grid, s);
    return launch_nc<8>(P, sample, i64, grid, s);
}

cudaError_t launch_finalize(const FinParams &F, cudaStream_t s) {
    const uint32_t blocks = F.njobs + F.hll_blocks;
    if (blocks) {
        fin_prefix<<<blocks, 1024, 0, s>>>(F);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint32_t outs = 1 + F.npreds + F.npairs;
    fin_output<<<(outs + 255) / 256, 256, 0, s>>>(F);
    return cudaGetLastError();
}

cudaError_t launch_minmax(const void *col, int dtype, uint64_t n, long long *mm, int sms, cudaStream_t s) {
    const uint64_t want = (n + 255) / 256;
    const int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
    minmax_kernel<<<grid, 256, 0, s>>>(col, dtype, n, mm);
    return cudaGetLastError();
}

cudaError_t launch_sample_mask(uint64_t nrows, uint64_t row0, uint64_t seed, uint64_t thr, bool all,
                               unsigned long long *bits, cudaStream_t s) {
    const uint64_t words = (nrows + 63) / 64;
    if (!words) return cudaSuccess;
    sample_mask_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(nrows, row0, seed, thr, all, bits);
    return cudaGetLastError();
}

}  // namespace gace
