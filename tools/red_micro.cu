// red_micro.cu — L2 atomic (red) throughput for random updates: 32- vs 64-bit, region size,
// and shared-memory atomics, to size the counter-update roof (SURVEY.md §8(d) roof 3).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o red_micro red_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint64_t i) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z ^= z >> 31;
    z *= 0xBF58476D1CE4E5B9ULL;
    return (uint32_t)(z >> 32);
}

template <int W>
__global__ void k_red(void *base, uint32_t mask, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t j = hsh(i) & mask;
        if (W == 4) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"((uint32_t *)base + j) : "memory");
        else asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"((uint64_t *)base + j) : "memory");
    }
}

__global__ void k_smem(uint32_t mask, uint64_t n, int *out) {
    extern __shared__ int sm[];
    for (int i = threadIdx.x; i <= (int)mask; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) atomicAdd(&sm[hsh(i) & mask], 1);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

int main() {
    void *buf;
    int *o;
    cudaMalloc(&buf, 1ULL << 30);
    cudaMalloc(&o, 4096 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint64_t n = 200000000ULL;
    float ms;
    for (uint32_t bytes : {1u << 22, 1u << 23, 1u << 26, 1u << 29}) {
        for (int w : {4, 8}) {
            const uint32_t mask = bytes / w - 1;
            for (int r = 0; r < 2; ++r) {
                cudaEventRecord(e0);
                if (w == 4) k_red<4><<<148 * 8, 512>>>(buf, mask, n);
                else k_red<8><<<148 * 8, 512>>>(buf, mask, n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            cudaEventElapsedTime(&ms, e0, e1);
            printf("red.u%-2d region %8u KB : %.3f ms  %.1f G/s\n", w * 8, bytes >> 10, ms, n / ms / 1e6);
        }
    }
    for (uint32_t words : {1024u, 5120u, 20480u, 40960u}) {
        cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            k_smem<<<148 * 2, 512, words * 4>>>(words - 1 < 1023 ? 1023 : (1u << (31 - __builtin_clz(words))) - 1, n, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("smem atomicAdd %6u words : %.3f ms  %.1f G/s  %s\n", words, ms, n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
