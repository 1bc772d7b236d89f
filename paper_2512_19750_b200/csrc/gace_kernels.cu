#include <algorithm>
// gace_kernels.cu -- sm_100a kernels of the GACE selectivity probe.
//
// probe_kernel (device code in gace_probe.cuh) streams every probed key column once
// from HBM and accumulates, in shared memory, per-column bucket histograms (-> counts
// by prefix differences), per-column-pair 2-D sub-bucket grids (-> joint counts by
// rectangle sums) and u32 HyperLogLog registers; each CTA adds its nonzero bins into
// global u64 accumulators and writes its registers as a per-CTA u8 partial.
// fin_prefix / fin_output turn the accumulators into the packed result
// [n_sampled, counts, joints] + registers.  No tensor cores: this is an HBM-bound
// integer scan.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>


#include "gace_kernels.h"
#include "gace_plan.h"
#include "gace_probe.cuh"

namespace gace {

// Generic probe kernels: only NC / SAMPLE / I64 are compile-time (gace_probe.cuh RtShape).
template <int NC, bool SAMPLE, bool I64>
__global__ void __launch_bounds__(kThreads, 1) probe_kernel(const __grid_constant__ ProbeParams P) {
    probe_body<RtShape<NC, SAMPLE, I64>>(P);
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

constexpr uint32_t kFinSatSmem = 5632;     // u64 cells of a summed-area table done in shared memory
constexpr uint32_t kFinHllWords = 64;      // register words per HLL merge block

// Programmatic dependent launch: the finalize kernels are launched with programmatic stream
// serialisation, so their launch overlaps the previous kernel's tail; each waits here for
// the previous grid to complete (no early trigger: its writes are all visible) before
// touching anything it produced.  A no-op when launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(1024) fin_prefix(const FinParams F) {
    __shared__ unsigned long long s_fin[kFinSatSmem];
    pdl_wait();
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
        } else if (J.na * J.nb <= kFinSatSmem) {   // JOB_SAT in shared memory (row, then column scans)
            const uint32_t na = J.na, nb = J.nb, st = nb + 1;
            unsigned long long *g = s_fin;
            for (uint32_t i = threadIdx.x; i < na * nb; i += blockDim.x) g[i] = src[i];
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < na; i += blockDim.x) {
                unsigned long long run = 0;
                for (uint32_t j = 0; j < nb; ++j) { run += g[i * nb + j]; g[i * nb + j] = run; }
            }
            __syncthreads();
            for (uint32_t j = threadIdx.x; j < nb; j += blockDim.x) {
                unsigned long long run = 0;
                for (uint32_t i = 0; i < na; ++i) { run += g[i * nb + j]; g[i * nb + j] = run; }
            }
            __syncthreads();
            for (uint32_t k = threadIdx.x; k < (na + 1) * st; k += blockDim.x) {   // zero border, stride nb + 1
                const uint32_t i = k / st, j = k - i * st;
                dst[k] = (i && j) ? g[(i - 1) * nb + j - 1] : 0ull;
            }
        } else {   // JOB_SAT too large for shared memory: in global memory
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
    } else {   // HLL: byte-wise max over the per-CTA partials, kFinHllWords words per block,
               // the partials split over blockDim.x / kFinHllWords slices, then a tree max
        const uint32_t words = F.hll_bytes / 4;
        const uint32_t w = (blockIdx.x - F.njobs) * kFinHllWords + threadIdx.x % kFinHllWords;
        const uint32_t sl = threadIdx.x / kFinHllWords, nsl = blockDim.x / kFinHllWords;
        const uint32_t *part = reinterpret_cast<const uint32_t *>(F.g_hll_part);
        uint32_t m = 0;
        if (w < words)
            for (uint32_t c = sl; c < F.nparts; c += nsl) m = __vmaxu4(m, part[(size_t)c * words + w]);
        uint32_t *r = reinterpret_cast<uint32_t *>(s_fin);
        r[threadIdx.x] = m;
        __syncthreads();
        for (uint32_t h = nsl / 2; h > 0; h /= 2) {
            if (sl < h) r[threadIdx.x] = __vmaxu4(r[threadIdx.x], r[threadIdx.x + h * kFinHllWords]);
            __syncthreads();
        }
        if (sl == 0 && w < words) reinterpret_cast<uint32_t *>(F.out_regs)[w] = r[threadIdx.x];
    }
}

__global__ void __launch_bounds__(1024) fin_bitmap_hll(const FinParams F) {
    __shared__ uint32_t R[kHllM];
    pdl_wait();
    const FinParams::BmJob J = F.bm[blockIdx.x];
    for (uint32_t i = threadIdx.x; i < kHllM; i += blockDim.x) R[i] = 0;
    __syncthreads();
    const uint32_t *bm = F.g_bm + J.goff;
    for (uint32_t i = threadIdx.x; i < J.words; i += blockDim.x) {
        uint32_t w = bm[i];
        while (w) {
            const uint32_t b = __ffs(w) - 1;
            w &= w - 1;
            uint32_t h = static_cast<uint32_t>(J.base + 32ll * i + b);
            h ^= h >> 16;
            h *= 0x85EBCA6BU;
            h ^= h >> 13;
            h *= 0xC2B2AE35U;
            h ^= h >> 16;
            atomicMax(R + (h >> (32 - kHllP)), __clz((h << kHllP) | (1u << (kHllP - 1))) + 1);
        }
    }
    __syncthreads();
    uint8_t *out = F.out_regs + (size_t)J.out * kHllM;
    for (uint32_t i = threadIdx.x; i < kHllM; i += blockDim.x) out[i] = (uint8_t)R[i];
}

// count of buckets [lo, hi] from a bucket-count prefix P(b) = pre[b * stride]
__device__ __forceinline__ unsigned long long iv(const unsigned long long *pre, uint32_t stride, uint32_t lo,
                                                 uint32_t hi) {
    return lo <= hi ? pre[(size_t)(hi + 1) * stride] - pre[(size_t)lo * stride] : 0ull;
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
    pdl_wait();
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long n = *F.g_nsamp;
    if (t == 0) F.out[0] = n;
    if (t >= 1 && t <= F.npreds) {
        const FinPred p = F.preds[t - 1];
        const unsigned long long c = iv(F.g_pre + p.pre, p.stride, p.lo, p.hi);
        F.out[t] = p.neg ? n - c : c;
    } else if (t > F.npreds && t <= F.npreds + F.npairs) {
        const FinPair q = F.pairs[t - 1 - F.npreds];
        unsigned long long r;
        if (q.kind == PAIR_DIRECT) {
            r = F.g_acc[q.pre];
        } else if (q.kind == PAIR_SAME) {
            const unsigned long long *pre = F.g_pre + q.pre;
            const uint32_t lo = max(q.li, q.lj), hi = min(q.hi, q.hj);
            r = combine(n, iv(pre, q.stride, q.li, q.hi), iv(pre, q.stride, q.lj, q.hj), iv(pre, q.stride, lo, hi),
                        q.negi, q.negj);
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
    // the other accumulator buffer (unused by this call) -> zero for the next call
    for (uint64_t i = t; i < F.zero_vec; i += (uint64_t)gridDim.x * blockDim.x) F.zero[i] = make_uint4(0u, 0u, 0u, 0u);
}

// ------------------------------------------------------------------ attach / test hook

// Attach-time column statistics: mm[0] = min, mm[1] = max, mm[2] = number of aligned row
// quads (rows 4q..4q+3) whose four keys are equal (clustered columns, e.g. a sorted key
// with repeats: the specialised probe then resolves such a quad once).
__global__ void minmax_kernel(const void *col, int dtype, uint64_t n, long long *mm) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    unsigned long long eq = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t nq = (n + 3) / 4;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
        long long v[4];
        const uint32_t cnt = n - 4 * q >= 4 ? 4u : (uint32_t)(n - 4 * q);
        for (uint32_t k = 0; k < 4; ++k) {
            const uint64_t i = 4 * q + (k < cnt ? k : 0);
            v[k] = dtype == 0 ? (long long)__ldg(static_cast<const int32_t *>(col) + i)
                              : __ldg(static_cast<const long long *>(col) + i);
            lo = min(lo, v[k]);
            hi = max(hi, v[k]);
        }
        eq += (cnt == 4 && v[0] == v[1] && v[1] == v[2] && v[2] == v[3]) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
        eq += __shfl_xor_sync(0xFFFFFFFFu, eq, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
        atomicAdd(reinterpret_cast<unsigned long long *>(mm + 2), eq);
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
    // the attribute is per device: set it for each device this instantiation runs on
    static std::mutex mu;
    static uint64_t configured = 0;      // bit d: device d done
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (dev >= 64 || !((configured >> dev) & 1ull)) {
            // the plan was budgeted with static_smem_reserve(SAMPLE): check the compiled kernel
            cudaFuncAttributes fa{};
            e = cudaFuncGetAttributes(&fa, k);
            if (e == cudaSuccess && fa.sharedSizeBytes > (size_t)static_smem_reserve(SAMPLE)) e = cudaErrorInvalidValue;
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kMaxSmem - static_smem_reserve(SAMPLE));
            if (e != cudaSuccess) {
                (void)cudaGetLastError();    // reported here; must not surface at the next launch
                return e;
            }
            if (dev < 64) configured |= 1ull << dev;
        }
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

template <class K>
static cudaError_t launch_pdl(K kern, unsigned blocks, unsigned threads, cudaStream_t s, const FinParams &F) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, F);
}

cudaError_t launch_finalize(const FinParams &F, cudaStream_t s) {
    const uint32_t blocks = F.njobs + F.hll_blocks;
    if (blocks) {
        cudaError_t e = launch_pdl(fin_prefix, blocks, 1024, s, F);
        if (e != cudaSuccess) return e;
    }
    if (F.nbm) {                         // after fin_prefix wrote the register blocks
        cudaError_t e = launch_pdl(fin_bitmap_hll, F.nbm, 1024, s, F);
        if (e != cudaSuccess) return e;
    }
    const uint32_t outs = 1 + F.npreds + F.npairs;
    const uint64_t zb = std::min<uint64_t>((F.zero_vec + 255) / 256, 296);
    return launch_pdl(fin_output, (unsigned)std::max<uint64_t>((outs + 255) / 256, zb), 256, s, F);
}

cudaError_t launch_minmax(const void *col, int dtype, uint64_t n, long long *mm, int sms, cudaStream_t s) {
    const uint64_t want = (n + 255) / 256;
    const int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
    minmax_kernel<<<grid, 256, 0, s>>>(col, dtype, n, mm);
    return cudaGetLastError();
}

// HLL register ceilings of one column (the largest rank any value of the domain
// [dl, dl + span] can put into each register; DESIGN.md §6 "HLL completion"): per-CTA
// shared maxima over a grid-stride range of the domain, merged into ce32 (u32[4096], zeroed
// by the caller) and packed to u8 by ceil_pack_kernel.  Hashes as in the probe (fmix32 for
// int32 columns, mix64(x + gamma) for int64).
__global__ void ceil_kernel(long long dl, unsigned long long span, int is64, uint32_t *ce32) {
    __shared__ uint32_t R[kHllM];
    for (uint32_t i = threadIdx.x; i < kHllM; i += blockDim.x) R[i] = 0;
    __syncthreads();
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long k = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; k <= span; k += stride) {
        const uint64_t v = (uint64_t)dl + k;
        uint32_t idx, r;
        if (!is64) {
            const uint32_t h = fmix32((uint32_t)v);
            idx = h >> (32 - kHllP);
            r = __clz((h << kHllP) | (1u << (kHllP - 1))) + 1;
        } else {
            const uint64_t h = mix64(v + GACE_GAMMA);
            idx = (uint32_t)(h >> (64 - kHllP));
            r = __clzll((h << kHllP) | (1ull << (kHllP - 1))) + 1;
        }
        if (r > R[idx]) atomicMax(&R[idx], r);
        if (k + stride < k) break;       // span near 2^64: no wrap-around
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kHllM; i += blockDim.x)
        if (R[i]) atomicMax(ce32 + i, R[i]);
}

__global__ void ceil_pack_kernel(const uint32_t *ce32, uint8_t *ce8) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kHllM) ce8[i] = (uint8_t)ce32[i];
}

cudaError_t launch_hll_ceilings(long long dl, unsigned long long span, bool is64, uint32_t *scratch32,
                                uint8_t *out8, int sms, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(scratch32, 0, 4 * kHllM, s);
    if (e != cudaSuccess) return e;
    const unsigned long long want = span / 1024 + 1;
    const unsigned grid = (unsigned)(want < (unsigned long long)sms * 2 ? want : (unsigned long long)sms * 2);
    ceil_kernel<<<grid, 1024, 0, s>>>(dl, span, is64 ? 1 : 0, scratch32);
    ceil_pack_kernel<<<kHllM / 256, 256, 0, s>>>(scratch32, out8);
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
