// gather_micro.cu — DRAM bytes fetched per sparse 8-byte gather, by load flavour.
// Each thread takes a block of 32 consecutive int64 rows of a 16 GB array and loads
// the rows whose hash bit says "survivor" (~5%), like the C4 key gathers.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_micro gather_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ bool survives(uint64_t i) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z ^= z >> 29;
    z *= 0xBF58476D1CE4E5B9ULL;
    return (z >> 40) % 1000 < 50;
}

template <int MODE>
__global__ void k_gather(const long long *__restrict__ a, uint64_t n, unsigned long long *out) {
    extern __shared__ long long sm[];
    unsigned long long acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 32;
    int q = 0;
    for (uint64_t base = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 32; base < n; base += stride) {
        for (int j = 0; j < 32; ++j) {
            const uint64_t i = base + j;
            if (!survives(i)) continue;
            long long v;
            if (MODE == 0) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(&sm[threadIdx.x * 4 + (q & 3)])), "l"(a + i));
                ++q;
                v = 0;
            } else if (MODE == 1) {
                asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(a + i));
            } else if (MODE == 2) {
                asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(a + i));
            } else if (MODE == 3) {
                asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(a + i));
            } else {
                asm volatile("ld.global.lu.b64 %0, [%1];" : "=l"(v) : "l"(a + i));
            }
            acc += v;
        }
    }
    if (MODE == 0) asm volatile("cp.async.wait_all;");
    if (acc == 42) out[0] = acc;
}

int main() {
    const uint64_t n = 2ULL << 30;   // 2^31 int64 = 16 GB
    long long *a;
    unsigned long long *o;
    if (cudaMalloc(&a, n * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&o, 8);
    cudaMemset(a, 1, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    uint64_t surv = 0;
    const char *names[] = {"cp.async.ca 8B", "ld.nc.L1::no_allocate", "ld.cg", "ld.nc.L2::64B", "ld.lu"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: k_gather<0><<<148 * 4, 256, 256 * 32>>>(a, n, o); break;
                case 1: k_gather<1><<<148 * 4, 256>>>(a, n, o); break;
                case 2: k_gather<2><<<148 * 4, 256>>>(a, n, o); break;
                case 3: k_gather<3><<<148 * 4, 256>>>(a, n, o); break;
                default: k_gather<4><<<148 * 4, 256>>>(a, n, o); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 1) printf("%-26s %8.3f ms\n", names[mode], ms);
        }
    }
    (void)surv;
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
