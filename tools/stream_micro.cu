// stream_micro.cu — read bandwidth of 3 int32 columns (C4's predicate columns, 12 GB):
// LDG.128 grid-stride vs a TMA-bulk smem ring (1 producer + N consumer warps).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o stream_micro stream_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void k_ldg(const int4 *a, const int4 *b, const int4 *c, uint64_t n4, int *out) {
    int acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        int4 v[12];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v[u * 3 + 0] = __ldg(a + i + u * stride);
            v[u * 3 + 1] = __ldg(b + i + u * stride);
            v[u * 3 + 2] = __ldg(c + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < 12; ++u) acc += (v[u].x < 368) + (v[u].y < 368) + (v[u].z < 368) + (v[u].w < 368);
    }
    for (; i < n4; i += stride) {
        int4 x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i);
        acc += x.x + y.y + z.z;
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

// TMA ring: tile = T rows per column, S stages, W consumer warps
__global__ void k_tma(const int *a, const int *b, const int *c, uint64_t n, int T, int S, int *out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 16;
    unsigned char *ring = smem + 256;
    const int W = blockDim.x / 32 - 1;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t stage = 3u * T * 4u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], W); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t tiles = n / T;
    if (warp == W) {
        if (lane == 0) {
            uint32_t i = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
                const uint32_t s = i % S;
                if (i >= (uint32_t)S) mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
                mbar_arrive_tx(&full[s], stage);
                unsigned char *d = ring + s * stage;
                bulk_g2s(d, a + t * T, T * 4, &full[s]);
                bulk_g2s(d + T * 4, b + t * T, T * 4, &full[s]);
                bulk_g2s(d + 2 * T * 4, c + t * T, T * 4, &full[s]);
            }
        }
        return;
    }
    int acc = 0;
    uint32_t i = 0;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const uint32_t s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        const int4 *d = reinterpret_cast<const int4 *>(ring + s * stage);
        for (int j = warp * 32 + lane; j < 3 * T / 4; j += W * 32) {
            int4 v = d[j];
            acc += (v.x < 368) + (v.y < 368) + (v.z < 368) + (v.w < 368);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

int main() {
    const uint64_t n = 1000000000ULL;
    int *a, *b, *c, *o;
    cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4); cudaMalloc(&o, 4);
    cudaMemset(a, 1, n * 4); cudaMemset(b, 2, n * 4); cudaMemset(c, 3, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int blocks : {148 * 2, 148 * 4, 148 * 8}) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            k_ldg<<<blocks, 512>>>((const int4 *)a, (const int4 *)b, (const int4 *)c, n / 4, o);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ldg   blocks=%5d            %.3f ms  %.0f GB/s\n", blocks, ms, 12e9 / ms / 1e6);
    }
    int cfg[][4] = {{2048, 4, 16, 1}, {2048, 6, 16, 1}, {2048, 8, 16, 1}, {4096, 4, 16, 1}, {4096, 3, 16, 1},
                    {8192, 2, 16, 1}, {2048, 4, 8, 2}, {1024, 8, 8, 2}, {2048, 3, 4, 3}};
    for (auto &k : cfg) {
        const int T = k[0], S = k[1], W = k[2], occ = k[3];
        const int smem = 256 + S * 3 * T * 4;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            k_tma<<<148 * occ, (W + 1) * 32, smem>>>(a, b, c, n, T, S, o);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tma   T=%5d S=%d W=%2d occ=%d smem=%6d  %.3f ms  %.0f GB/s  %s\n", T, S, W, occ, smem, ms, 12e9 / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
