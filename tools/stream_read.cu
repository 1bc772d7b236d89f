// Read-only streaming ceiling of this B200 ("a read-only streaming
// microbenchmark run on the box" -- the third roofline denominator next to the measured
// copy peak and the nominal 8 TB/s).
//
// Reads the C5 layout -- 4 int32 columns of 600,037,902 rows, 9.6006 GB, each key once --
// with a live reduction (XOR of every key, stored per CTA so nothing is dead code), in
// the access patterns the probe kernels can use:
//   ldg        one 128-bit non-allocating load per column per thread and iteration,
//              persistent grid of 148 x B CTAs (the probe's pattern without its work)
//   ldg_pf     the same plus an L2 prefetch two iterations ahead (the probe's prefetch)
//   ldg_x2     two units per thread and iteration (twice the loads in flight)
//   bulk       cp.async.bulk (TMA 1-D bulk copy, SASS UBLKCP) global -> shared through a
//              4-stage mbarrier ring per CTA; one elected thread issues, all threads reduce
// Output: one JSON line per variant and configuration (best / median of the timed reps,
// CUDA events on the launching stream, 3 warm-up launches; the inputs are 76x L2).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o build/stream_read tools/stream_read.cu
//   build/stream_read [rows] [reps]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int NC = 4;
struct Cols {
    const int *c[NC];
    uint64_t nunits;      // 16-byte units per column
};

__device__ __forceinline__ int4 ld_stream(const void *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <int PF, int X2>
__global__ void __launch_bounds__(1024) k_ldg(Cols C, uint32_t *out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (X2) {
        for (; u + stride < C.nunits; u += 2 * stride) {
            int4 a[NC], b[NC];
#pragma unroll
            for (int s = 0; s < NC; ++s) {
                a[s] = ld_stream(C.c[s] + 4 * u);
                b[s] = ld_stream(C.c[s] + 4 * (u + stride));
            }
#pragma unroll
            for (int s = 0; s < NC; ++s) acc ^= a[s].x ^ a[s].y ^ a[s].z ^ a[s].w ^ b[s].x ^ b[s].y ^ b[s].z ^ b[s].w;
        }
    }
    for (; u < C.nunits; u += stride) {
        if (PF && u + 2 * stride < C.nunits) {
#pragma unroll
            for (int s = 0; s < NC; ++s) asm volatile("prefetch.global.L2 [%0];" ::"l"(C.c[s] + 4 * (u + 2 * stride)));
        }
        int4 a[NC];
#pragma unroll
        for (int s = 0; s < NC; ++s) a[s] = ld_stream(C.c[s] + 4 * u);
#pragma unroll
        for (int s = 0; s < NC; ++s) acc ^= a[s].x ^ a[s].y ^ a[s].z ^ a[s].w;
    }
    acc = __reduce_xor_sync(0xFFFFFFFFu, acc);
    if ((threadIdx.x & 31) == 0) atomicXor(out + blockIdx.x, acc);
}

// ---- cp.async.bulk ring: CTA-contiguous spans of every column, chunk = kChunk bytes per column
constexpr int kStages = 4;
constexpr uint32_t kChunk = 8192;          // bytes per column per stage (4 columns: 32 KB a stage)

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512) k_bulk(Cols C, uint32_t *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[kStages];
    const uint64_t bytes = C.nunits * 16;
    const uint64_t nchunks = (bytes + kChunk - 1) / kChunk;
    // chunks k = blockIdx.x, blockIdx.x + gridDim.x, ...
    const uint64_t first = blockIdx.x, step = gridDim.x;
    const uint64_t mine = first < nchunks ? (nchunks - first + step - 1) / step : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](uint64_t j) {            // j-th chunk of this CTA into stage j % kStages
        const uint64_t k = first + j * step;
        const uint64_t off = k * kChunk;
        const uint32_t n = (uint32_t)umin64(kChunk, bytes - off);
        const int st = (int)(j % kStages);
        const uint32_t bar = smem_u32(&full[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(n * NC));
        for (int s = 0; s < NC; ++s) {
            const uint32_t dst = smem_u32(sm + (st * NC + s) * kChunk);
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "l"(reinterpret_cast<const char *>(C.c[s]) + off), "r"(n), "r"(bar)
                         : "memory");
        }
    };
    if (threadIdx.x == 0)
        for (uint64_t j = 0; j < umin64(kStages, mine); ++j) issue(j);
    uint32_t acc = 0;
    for (uint64_t j = 0; j < mine; ++j) {
        const int st = (int)(j % kStages);
        const uint32_t parity = (uint32_t)((j / kStages) & 1);
        const uint32_t bar = smem_u32(&full[st]);
        asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}"
                     ::"r"(bar), "r"(parity) : "memory");
        const uint64_t off = (first + j * step) * kChunk;
        const uint32_t n = (uint32_t)umin64(kChunk, bytes - off);
        for (int s = 0; s < NC; ++s) {
            const int4 *p = reinterpret_cast<const int4 *>(sm + (st * NC + s) * kChunk);
            for (uint32_t i = threadIdx.x; i < n / 16; i += blockDim.x) {
                const int4 v = p[i];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
        }
        __syncthreads();                      // stage consumed by every thread
        if (threadIdx.x == 0 && j + kStages < mine) issue(j + kStages);
    }
    acc = __reduce_xor_sync(0xFFFFFFFFu, acc);
    if ((threadIdx.x & 31) == 0) atomicXor(out + blockIdx.x, acc);
}

static void report(const char *name, int grid, int block, double bytes, std::vector<float> &ms, uint32_t check) {
    std::sort(ms.begin(), ms.end());
    const double best = ms.front(), med = ms[ms.size() / 2];
    printf("{\"variant\": \"%s\", \"grid\": %d, \"block\": %d, \"bytes\": %.0f, \"best_ms\": %.4f, \"median_ms\": %.4f, "
           "\"best_gbs\": %.1f, \"median_gbs\": %.1f, \"xor\": %u}\n",
           name, grid, block, bytes, best, med, bytes / (best * 1e-3) / 1e9, bytes / (med * 1e-3) / 1e9, check);
    fflush(stdout);
}

int main(int argc, char **argv) {
    const uint64_t rows = argc > 1 ? strtoull(argv[1], nullptr, 10) : 600037902ull;
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t nunits = rows / 4;                      // whole 16-byte units (tail ignored)
    const double bytes = (double)nunits * 16 * NC;
    Cols C{};
    C.nunits = nunits;
    for (int s = 0; s < NC; ++s) {
        int *p = nullptr;
        CK(cudaMalloc(&p, nunits * 16));
        CK(cudaMemset(p, 0x11 * (s + 1), nunits * 16));
        C.c[s] = p;
    }
    uint32_t *out = nullptr;
    CK(cudaMalloc(&out, 4096 * 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](const char *name, auto launch, int grid, int block) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        std::vector<float> ms;
        for (int r = 0; r < reps; ++r) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float t = 0;
            CK(cudaEventElapsedTime(&t, e0, e1));
            ms.push_back(t);
        }
        CK(cudaGetLastError());
        uint32_t h[1] = {0};
        CK(cudaMemcpy(h, out, 4, cudaMemcpyDeviceToHost));
        report(name, grid, block, bytes, ms, h[0]);
    };
    for (int bps : {1, 2}) {
        const int grid = sms * bps, block = 1024 / bps;
        run("ldg", [&] { k_ldg<0, 0><<<grid, block>>>(C, out); }, grid, block);
        run("ldg_pf", [&] { k_ldg<1, 0><<<grid, block>>>(C, out); }, grid, block);
        run("ldg_x2", [&] { k_ldg<0, 1><<<grid, block>>>(C, out); }, grid, block);
    }
    {
        const size_t smem = (size_t)kStages * NC * kChunk;
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        for (int bps : {1, 2}) {
            const int grid = sms * bps;
            run("bulk", [&] { k_bulk<<<grid, 512, smem>>>(C, out); }, grid, 512);
        }
    }
    return 0;
}
