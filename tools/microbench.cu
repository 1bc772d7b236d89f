// Shared-memory update throughput on this GPU (design input for the probe's counters).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0: atomicAdd random bucket of NB; 1: atomicAdd same address; 2: atomicAdd lane-distinct banks;
// 3: private byte counters (LDS.U8/STS.U8, thread-private region); 4: LDS random (read only);
// 5: atomicAdd random bucket, per-warp private copy of the histogram
template <int MODE>
__global__ void k_smem(int iters, int nb, uint32_t smem_words, uint32_t *out) {
    extern __shared__ uint32_t sm[];
    const int tid = threadIdx.x;
    for (uint32_t i = tid; i < smem_words; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    uint32_t x = hash32(blockIdx.x * 4096 + tid);
    uint32_t acc = 0;
    uint8_t *sm8 = reinterpret_cast<uint8_t *>(sm);
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t b = (x >> 8) % nb;
        if (MODE == 0) atomicAdd(sm + b, 1u);
        if (MODE == 1) atomicAdd(sm + 7, 1u);
        if (MODE == 2) atomicAdd(sm + (tid & 31) + 32 * (it & 7), 1u);
        if (MODE == 3) { uint8_t *p = sm8 + b * blockDim.x + tid; *p = *p + 1; }
        if (MODE == 4) acc += sm[b];
        if (MODE == 5) atomicAdd(sm + (tid >> 5) * nb + b, 1u);
    }
    if (acc == 0x12345678) out[0] = acc;
}

template <int MODE>
float run(int nb, int threads, int iters, size_t smem) {
    cudaFuncSetAttribute(k_smem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    uint32_t *out;
    cudaMalloc(&out, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k_smem<MODE><<<sms, threads, smem>>>(iters, nb, (uint32_t)(smem / 4), out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_smem<MODE><<<sms, threads, smem>>>(iters, nb, (uint32_t)(smem / 4), out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    cudaFree(out);
    // lane-ops per SM per ns
    return (float)threads * iters / (ms * 1e6f);
}

int main() {
    const int it = 4096;
    printf("lane-updates per SM per ns (x1.965 GHz -> per cycle: divide by 1.965)\n");
    for (int nb : {129, 1025}) {
        printf("nb=%d atomic random        : %.2f\n", nb, run<0>(nb, 1024, it, 64 * 1024));
        printf("nb=%d atomic per-warp hist : %.2f\n", nb, run<5>(nb, 1024, it, 32 * nb * 4 > 200 * 1024 ? 200 * 1024 : 32 * nb * 4 + 64));
        printf("nb=%d private u8 (128 thr) : %.2f\n", nb, run<3>(nb, 128, it, nb * 128 + 64));
        printf("nb=%d lds random           : %.2f\n", nb, run<4>(nb, 1024, it, 64 * 1024));
    }
    printf("atomic same address     : %.2f\n", run<1>(129, 1024, it / 4, 64 * 1024));
    printf("atomic distinct banks   : %.2f\n", run<2>(129, 1024, it, 64 * 1024));
    return 0;
}
