// Shared-memory access throughput on this GPU (design input for the probe's tables/counters).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu && build/microbench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// Each thread performs `iters` accesses at pseudo-random word indices in [0, nwords).
// MODE 0: atomicAdd(+1)          (compiles to ATOMS.POPC.INC)
// MODE 1: atomicAdd(+v), v reg   (ATOMS.ADD)
// MODE 2: LDS.32   3: LDS.64   4: LDS.128 (entry index random, 16-B aligned)
// MODE 5: atomicMax(+v)          6: LDS.32 all lanes of a warp same address (broadcast)
template <int MODE>
__global__ void k_smem(int iters, uint32_t nwords, uint32_t smem_words, uint32_t *out) {
    extern __shared__ uint32_t sm[];
    const int tid = threadIdx.x;
    for (uint32_t i = tid; i < smem_words; i += blockDim.x) sm[i] = i;
    __syncthreads();
    uint32_t x = hash32(blockIdx.x * 4096 + tid);
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t b = (x >> 8) % nwords;
        if (MODE == 0) atomicAdd(sm + b, 1u);
        if (MODE == 1) atomicAdd(sm + b, (x & 1) + 1);
        if (MODE == 2) acc += sm[b];
        if (MODE == 3) { const uint2 v = reinterpret_cast<const uint2 *>(sm)[b >> 1]; acc += v.x ^ v.y; }
        if (MODE == 4) { const uint4 v = reinterpret_cast<const uint4 *>(sm)[b >> 2]; acc += v.x ^ v.y ^ v.z ^ v.w; }
        if (MODE == 5) atomicMax(sm + b, x);
        if (MODE == 6) acc += sm[__shfl_sync(0xffffffffu, b, 0)];
    }
    if (acc == 0x12345678) out[0] = acc;
}

template <int MODE>
float run(uint32_t nwords, int threads, int iters) {
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(k_smem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint32_t *out;
    cudaMalloc(&out, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k_smem<MODE><<<sms, threads, smem>>>(iters, nwords, (uint32_t)(smem / 4), out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_smem<MODE><<<sms, threads, smem>>>(iters, nwords, (uint32_t)(smem / 4), out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    cudaFree(out);
    // SM-cycles per warp-instruction at 1.965 GHz
    const double warp_instr_per_sm = (double)threads / 32 * iters;
    return (float)(ms * 1e-3 * 1.965e9 / warp_instr_per_sm);
}

int main() {
    const int it = 4096;
    printf("SM cycles per warp-wide access (random word in a table of N words), 512 threads/SM\n");
    for (uint32_t n : {129u, 4257u, 16384u}) {
        printf("N=%5u  ATOMS.POPC.INC %.2f  ATOMS.ADD %.2f  ATOMS.MAX %.2f  LDS.32 %.2f  LDS.64 %.2f  LDS.128 %.2f  bcast %.2f\n", n,
               run<0>(n, 512, it), run<1>(n, 512, it), run<5>(n, 512, it), run<2>(n, 512, it), run<3>(n, 512, it),
               run<4>(n, 512, it), run<6>(n, 512, it));
    }
    return 0;
}
