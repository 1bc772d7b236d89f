// gace_sets.cu -- sm_100a kernel of the candidate-set probe (gace_probe_sets).
//
// PAPER.md §IV-H Exp. D (lines 250-270): per candidate set m, the number of sampled rows on
// which every member predicate holds.  One pass over the probed key columns (128-bit
// non-allocating loads, each key read once); per row and column one cell lookup (+ a short
// in-cell binary search on cells holding breakpoints) gives the bucket, and one shared-memory
// load gives that bucket's set-satisfaction mask (gace_sets.h); the AND over the columns is
// the row's set mask.  Counting: 5 bit-sliced planes per lane (a carry-save add per row),
// flushed every 28 rows by a 32x32 warp bit-matrix transpose (5 shuffles) + popcount, so the
// cost per row is independent of K and of M within a 32-set word, and there are no per-row
// atomics.  No tensor cores: an integer scan, not a contraction.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gace_sets.h"

namespace gace {
namespace {

__device__ __forceinline__ uint64_t sets_mix64(uint64_t z) {   // SplitMix64 finaliser (DESIGN.md §2 step 1)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ bool sets_keep(uint64_t seed, uint64_t thr, uint64_t g) {
    return sets_mix64(seed + (g + 1) * 0x9E3779B97F4A7C15ULL) < thr;
}

__device__ __forceinline__ int4 ld_nc128(const void *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Predicated 128-bit load into r (unchanged when !pred): one instruction, no register copies
__device__ __forceinline__ void ld_nc128_if(bool pred, const void *p, int4 &r) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n"
                 " @q ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%5];\n}"
                 : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
                 : "r"((uint32_t)pred), "l"(p));
}

// #{i < n : bps[i] <= u} over sorted bps (branch-free binary search)
__device__ __forceinline__ uint32_t count_le(const uint64_t *bps, uint32_t n, uint64_t u) {
    uint32_t lo = 0;
    while (n > 0) {
        const uint32_t half = n >> 1;
        const bool right = bps[lo + half] <= u;
        lo = right ? lo + half + 1 : lo;
        n = right ? n - half - 1 : half;
    }
    return lo;
}

// 32x32 bit-matrix transpose across the warp (recursive off-diagonal block swap):
// on return, bit l of lane m's word = bit m of lane l's input word.
__device__ __forceinline__ uint32_t warp_transpose(uint32_t x, uint32_t lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                           : s == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
        x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
    }
    return x;
}

template <int W>
__device__ __forceinline__ void flush(uint32_t (&pl)[W][5], uint32_t (&cnt)[W], uint32_t lane) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
        uint32_t acc = 0;
#pragma unroll
        for (int p = 0; p < 5; ++p) {
            acc += static_cast<uint32_t>(__popc(warp_transpose(pl[j][p], lane))) << p;
            pl[j][p] = 0u;
        }
        cnt[j] += acc;
    }
}

}  // namespace

// Keys of unit u of column c (4 rows) into r when pred (int64 columns: two 128-bit loads).
template <bool I64>
__device__ __forceinline__ void load_col(const SetsParams &P, int c, uint64_t u, int4 (&r)[I64 ? 2 : 1],
                                         bool pred = true) {
    const char *p = static_cast<const char *>(P.col[c].ptr);
    if (!(I64 && P.col[c].is64)) {
        ld_nc128_if(pred, p + u * 16, r[0]);
    } else {
        ld_nc128_if(pred, p + u * 32, r[0]);
        ld_nc128_if(pred, p + u * 32 + 16, r[I64 ? 1 : 0]);
    }
}

// Offsets u = v - dlo of the four keys in r.
template <bool I64>
__device__ __forceinline__ void offsets(const SetsCol &C, const int4 (&r)[I64 ? 2 : 1], uint64_t (&uo)[4]) {
    if (!(I64 && C.is64)) {
        const uint32_t d = static_cast<uint32_t>(C.dlo);
        uo[0] = static_cast<uint32_t>(r[0].x) - d;
        uo[1] = static_cast<uint32_t>(r[0].y) - d;
        uo[2] = static_cast<uint32_t>(r[0].z) - d;
        uo[3] = static_cast<uint32_t>(r[0].w) - d;
    } else {
        const int4 a = r[0], b = r[I64 ? 1 : 0];
        const uint64_t d = static_cast<uint64_t>(C.dlo);
        uo[0] = ((static_cast<uint64_t>(static_cast<uint32_t>(a.y)) << 32) | static_cast<uint32_t>(a.x)) - d;
        uo[1] = ((static_cast<uint64_t>(static_cast<uint32_t>(a.w)) << 32) | static_cast<uint32_t>(a.z)) - d;
        uo[2] = ((static_cast<uint64_t>(static_cast<uint32_t>(b.y)) << 32) | static_cast<uint32_t>(b.x)) - d;
        uo[3] = ((static_cast<uint64_t>(static_cast<uint32_t>(b.w)) << 32) | static_cast<uint32_t>(b.z)) - d;
    }
}

// AND the set-satisfaction masks of column c's four keys (offsets uo) into x[k].  FOLD (one 32-set word): a cell with no breakpoint inside holds its sat
// mask itself (bit 31 clear); other cells hold kSetsImpure | b0 | n << 20.  Otherwise a
// cell holds b0 | n << 20 and the mask is sat[b].  The in-cell search runs only for the
// keys in cells with breakpoints, behind one warp-level branch per column.
template <int W, bool FOLD, bool I64>
__device__ __forceinline__ void column_masks(const SetsCol &C, const uint32_t *sm32, const uint64_t *sm64,
                                             const uint64_t (&uo)[4], uint32_t (&x)[4][W]) {
    const bool w64 = I64 && C.is64;
    const uint32_t *cells = sm32 + C.cell_off;
    uint32_t cw[4], slow = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t cell = w64 ? static_cast<uint32_t>(uo[k] >> C.shift) : static_cast<uint32_t>(uo[k]) >> C.shift;
        cw[k] = cells[cell];
        if (FOLD) slow |= cw[k];
        else slow |= cw[k] >> kSetsCellB0Bits;
    }
    if (FOLD && !(slow & kSetsImpure)) {
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k][0] &= cw[k];
        return;
    }
    const uint64_t *bps = sm64 + C.bps_off;
    const uint32_t *sat = sm32 + C.sat_off;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t m = cw[k];                       // FOLD: a breakpoint-free cell's mask
        if (!FOLD || (cw[k] & kSetsImpure)) {
            uint32_t b = cw[k] & ((1u << kSetsCellB0Bits) - 1u);
            const uint32_t n = (cw[k] & ~kSetsImpure) >> kSetsCellB0Bits;
            if (n == 1) b += bps[b] <= uo[k] ? 1u : 0u;     // the common boundary cell
            else if (n) b += count_le(bps + b, n, uo[k]);
            if (FOLD) {
                m = sat[b];
            } else {
#pragma unroll
                for (int j = 0; j < W; ++j) x[k][j] &= sat[b * W + j];
            }
        }
        if (FOLD) x[k][0] &= m;
    }
}

template <int W>
__device__ __forceinline__ void csa_add(uint32_t (&pl)[W][5], const uint32_t (&x)[4][W]) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < W; ++j) {
            uint32_t cy = x[k][j];
#pragma unroll
            for (int p = 0; p < 5; ++p) {
                const uint32_t t = pl[j][p] & cy;
                pl[j][p] ^= cy;
                cy = t;
            }
        }
}

// One CTA per SM of 1024 threads; each thread owns units of 4 rows.  Column-streamed keys:
// once column c of the current unit is consumed, its registers are refilled with column c
// of the thread's next unit, so the next keys are in flight during the rest of the unit.
// NCM: column slots compiled; EXACT: ncols == NCM (no run-time column checks, which would
// otherwise make the compiler shuffle the streamed key registers between paths).
template <int W, int NCM, bool EXACT, bool I64, bool SAMPLE, bool FOLD>
__global__ void __launch_bounds__(kSetsThreads, 1) sets_kernel(const __grid_constant__ SetsParams P) {
    extern __shared__ uint4 s_img[];
    __shared__ uint32_t s_cnt[kSetsMaxWords * 32];
    for (uint32_t i = threadIdx.x; i < P.image_u4; i += blockDim.x) s_img[i] = __ldg(P.image + i);
    for (uint32_t i = threadIdx.x; i < W * 32; i += blockDim.x) s_cnt[i] = 0u;
    __syncthreads();
    const uint32_t *sm32 = reinterpret_cast<const uint32_t *>(s_img);
    const uint64_t *sm64 = reinterpret_cast<const uint64_t *>(s_img);

    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nfull = P.nrows / 4;
    const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t pl[W][5], cnt[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        cnt[j] = 0u;
#pragma unroll
        for (int p = 0; p < 5; ++p) pl[j][p] = 0u;
    }
    uint32_t kept = 0;
    int pend = 0;
    auto quad_keep = [&](uint64_t u) -> uint32_t {
        if (u >= nfull) return 0u;
        if (!SAMPLE) return 0xFu;
        const uint64_t g0 = P.row0 + 4 * u;
        uint32_t kk = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) kk |= (sets_keep(P.seed, P.thr, g0 + k) ? 1u : 0u) << k;
        return kk;
    };
    int4 r[NCM][I64 ? 2 : 1] = {};
    uint64_t u = gw * 32 + lane;
    uint32_t keep = quad_keep(u);
#pragma unroll
    for (int c = 0; c < NCM; ++c)
        if (EXACT || c < (int)P.ncols) load_col<I64>(P, c, u, r[c], keep != 0u);
    // warp-uniform trip count (the flush is warp-collective)
    for (uint64_t base = gw * 32; base < nfull; base += stride, u += stride) {
        const uint32_t keep_n = quad_keep(u + stride);
        kept += __popc(keep);
        uint32_t x[4][W];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < W; ++j) x[k][j] = ((keep >> k) & 1u) ? 0xFFFFFFFFu : 0u;
        if (keep) {
#pragma unroll
            for (int c = 0; c < NCM; ++c) {
                if (!EXACT && c >= (int)P.ncols) break;
                uint64_t uo[4];
                offsets<I64>(P.col[c], r[c], uo);
                load_col<I64>(P, c, u + stride, r[c], keep_n != 0u);
                column_masks<W, FOLD, I64>(P.col[c], sm32, sm64, uo, x);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NCM; ++c)
                if (EXACT || c < (int)P.ncols) load_col<I64>(P, c, u + stride, r[c], keep_n != 0u);
        }
        keep = keep_n;
        csa_add<W>(pl, x);
        pend += 4;
        if (pend >= 28) {
            flush<W>(pl, cnt, lane);
            pend = 0;
        }
    }
    // tail rows [4 * nfull, nrows): lanes 0..2 of global warp 0, one row each
    if (gw == 0 && 4 * nfull < P.nrows) {
        const uint64_t row = 4 * nfull + lane;
        uint32_t x[4][W];
        const bool mine = row < P.nrows && (!SAMPLE || sets_keep(P.seed, P.thr, P.row0 + row));
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < W; ++j) x[k][j] = (k == 0 && mine) ? 0xFFFFFFFFu : 0u;
        if (mine) {
            kept += 1;
            for (int c = 0; c < (int)P.ncols; ++c) {
                const SetsCol &C = P.col[c];
                uint64_t uo[4];
                if (I64 && C.is64) uo[0] = static_cast<uint64_t>(static_cast<const long long *>(C.ptr)[row]) - static_cast<uint64_t>(C.dlo);
                else uo[0] = static_cast<uint32_t>(static_cast<const int32_t *>(C.ptr)[row]) - static_cast<uint32_t>(C.dlo);
                uo[1] = uo[2] = uo[3] = uo[0];
                column_masks<W, FOLD, I64>(C, sm32, sm64, uo, x);
            }
        }
        csa_add<W>(pl, x);
        pend += 1;
    }
    if (pend) flush<W>(pl, cnt, lane);
#pragma unroll
    for (int j = 0; j < W; ++j)
        if (cnt[j]) atomicAdd(&s_cnt[j * 32 + lane], cnt[j]);
    kept = __reduce_add_sync(0xFFFFFFFFu, kept);
    if (lane == 0 && kept) atomicAdd(P.g_nsamp, (unsigned long long)kept);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < W * 32; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(P.g_counts + i, (unsigned long long)s_cnt[i]);
}

namespace {
template <int W, int NCM, bool EXACT, bool I64, bool SAMPLE>
cudaError_t launch_t(const SetsParams &P, int grid, size_t smem, cudaStream_t s) {
    auto k = P.fold ? sets_kernel<W, NCM, EXACT, I64, SAMPLE, W == 1> : sets_kernel<W, NCM, EXACT, I64, SAMPLE, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();        // reported here; must not surface at the next launch
        return e;
    }
    k<<<grid, kSetsThreads, smem, s>>>(P);
    return cudaGetLastError();
}

template <int W, int NCM, bool EXACT>
cudaError_t launch_w(const SetsParams &P, bool sample, bool i64, int grid, size_t smem, cudaStream_t s) {
    if (i64)
        return sample ? launch_t<W, NCM, EXACT, true, true>(P, grid, smem, s)
                      : launch_t<W, NCM, EXACT, true, false>(P, grid, smem, s);
    return sample ? launch_t<W, NCM, EXACT, false, true>(P, grid, smem, s)
                  : launch_t<W, NCM, EXACT, false, false>(P, grid, smem, s);
}

// exact column counts 1..4 for one or two 32-set words; run-time column counts otherwise
template <int W>
cudaError_t launch_nc(const SetsParams &P, bool sample, bool i64, int grid, size_t smem, cudaStream_t s) {
    if (W <= 2) {
        switch (P.ncols) {
            case 1: return launch_w<W, 1, true>(P, sample, i64, grid, smem, s);
            case 2: return launch_w<W, 2, true>(P, sample, i64, grid, smem, s);
            case 3: return launch_w<W, 3, true>(P, sample, i64, grid, smem, s);
            case 4: return launch_w<W, 4, true>(P, sample, i64, grid, smem, s);
            default: break;
        }
    }
    return P.ncols <= 4 ? launch_w<W, 4, false>(P, sample, i64, grid, smem, s)
                        : launch_w<W, 8, false>(P, sample, i64, grid, smem, s);
}
}  // namespace

cudaError_t launch_sets(const SetsParams &P, bool sample, bool i64, int grid, cudaStream_t s) {
    const size_t smem = 16ull * P.image_u4;
    switch (P.W) {
        case 1: return launch_nc<1>(P, sample, i64, grid, smem, s);
        case 2: return launch_nc<2>(P, sample, i64, grid, smem, s);
        case 4: return launch_nc<4>(P, sample, i64, grid, smem, s);
        case 8: return launch_nc<8>(P, sample, i64, grid, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gace
