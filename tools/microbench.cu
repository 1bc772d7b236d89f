// Shared-memory access throughput on this GPU (design input for the probe's tables and
// counters): SM cycles per warp-wide access, for random / conflict-free / broadcast
// addresses, loads and atomics.  Addresses come from registers with two ALU ops per
// access, so the shared-memory pipe (not the ALU) is what is measured.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu && build/microbench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// MODE 0 LDS.32 random   1 ATOMS.ADD random   2 ATOMS.MAX random   3 LDS.32 broadcast
//      4 LDS.32 conflict-free   5 ATOMS.ADD conflict-free   6 LDS.128 random
//      7 RED.ADD random (no return, asm)   8 LDS.U16 random
template <int MODE>
__global__ void k_smem(int iters, uint32_t mask, uint32_t *out) {
    extern __shared__ uint32_t sm[];
    for (uint32_t i = threadIdx.x; i <= mask + 4; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t off[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        uint32_t r = hash32(blockIdx.x * 65536 + threadIdx.x * 8 + j);
        if (MODE == 3) r = hash32(blockIdx.x * 65536 + (threadIdx.x >> 5) * 8 + j);
        if (MODE == 4 || MODE == 5) r = (r & ~31u) | lane;
        off[j] = r;
    }
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        const uint32_t step = (uint32_t)it * 0x9E3779B9u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t a = (off[j] + (MODE == 4 || MODE == 5 ? (step & ~31u) : step)) & mask;
            if (MODE == 6) a &= ~3u;
            if (MODE == 0 || MODE == 3 || MODE == 4) acc += sm[a];
            if (MODE == 1 || MODE == 5) atomicAdd(sm + a, 1u);
            if (MODE == 2) atomicMax(sm + a, a);
            if (MODE == 6) { const uint4 v = *reinterpret_cast<const uint4 *>(sm + a); acc += v.x ^ v.w; }
            if (MODE == 7)
                asm volatile("red.shared.add.u32 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(sm + a)) : "memory");
            if (MODE == 8) acc += reinterpret_cast<const uint16_t *>(sm)[a];
        }
    }
    if (acc == 0x12345678) out[0] = acc;
}

template <int MODE>
float run(uint32_t words, int threads, int iters) {
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(k_smem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint32_t *out;
    cudaMalloc(&out, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k_smem<MODE><<<sms, threads, smem>>>(iters, words - 1, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_smem<MODE><<<sms, threads, smem>>>(iters, words - 1, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    cudaFree(out);
    const double warp_instr_per_sm = (double)threads / 32 * iters * 8;
    return (float)(ms * 1e-3 * 1.965e9 / warp_instr_per_sm);   // SM cycles per warp access (at max clock)
}

int main() {
    const int it = 2048;
    for (int threads : {512, 1024}) {
        printf("SM cycles per warp-wide access, %d threads/SM (1 CTA)\n", threads);
        for (uint32_t n : {256u, 4096u, 16384u}) {
            printf("N=%5u  LDS.32 rand %.2f  LDS.U16 rand %.2f  LDS.128 rand %.2f  ATOMS.ADD rand %.2f  RED.ADD rand %.2f  "
                   "ATOMS.MAX rand %.2f  LDS bcast %.2f  LDS cfree %.2f  ATOMS cfree %.2f\n", n,
                   run<0>(n, threads, it), run<8>(n, threads, it), run<6>(n, threads, it), run<1>(n, threads, it),
                   run<7>(n, threads, it), run<2>(n, threads, it), run<3>(n, threads, it), run<4>(n, threads, it),
                   run<5>(n, threads, it));
        }
    }
    return 0;
}
