// zerocopy_micro.cu — sparse 8-byte gathers from pinned host memory over PCIe (UVA), at ~5%
// of rows (the C4 survivor pattern), vs a bulk H2D copy of the same array.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/zerocopy_micro tools/zerocopy_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ bool survives(uint64_t i) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z ^= z >> 29;
    z *= 0xBF58476D1CE4E5B9ULL;
    return (z >> 40) % 1000 < 50;
}

__global__ void k_gather(const long long *a, uint64_t n, unsigned long long *out) {
    unsigned long long acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        if (survives(i)) acc += a[i];
    if (acc == 42) out[0] = acc;
}

int main() {
    const uint64_t n = 1ULL << 29;   // 4 GB of int64
    long long *h, *d;
    unsigned long long *o;
    cudaHostAlloc(&h, n * 8, cudaHostAllocMapped);
    for (uint64_t i = 0; i < n; i += 512) h[i] = 1;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bulk H2D 4 GB: %.2f ms  %.1f GB/s\n", ms, n * 8 / ms / 1e6);
    for (int grid : {148 * 4, 148 * 16, 148 * 64}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_gather<<<grid, 256>>>(h, n, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        const double req = n * 0.05;
        printf("zero-copy 5%% gathers grid %5d: %.2f ms  %.1f M req/s  (bulk-equivalent %.1f GB/s)  %s\n", grid, ms,
               req / ms / 1e3, n * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
