// roofs_micro.cu — the three roofs of SURVEY.md §8(d), measured on this B200, written as
// one JSON object (MEASURED_ROOFS.json):
//   read_stream_gbs  : read-only stream of 12 GB with 128-bit loads (HBM roof, read side;
//                      the copy figure of MEASURED_PEAKS.json counts read + write)
//   hash_*           : roof 2, the integer pipe: the exact xi/h sequence of the scan
//                      (csrc/hash.cuh: degree-3 xi + degree-1 h, mod 2^61-1) per (key, row),
//                      narrow path (keys < 2^32, 64x32 lazy Horner) and wide path (64x64);
//                      reported in (key, row) hash pairs per second
//   atoms_*          : roof 3, counter updates: shared-memory int32 atomicAdd (privatised
//                      sketches, 20 KB = d 5 x w 1024 region) and L2 red.add (u32 over a 4 MB
//                      histogram, u64 over a 10.5 MB matrix sketch), random addresses
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2102_02440_b200/csrc \
//            -o tools/roofs_micro tools/roofs_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "hash.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t i) {
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z ^= z >> 31;
    z *= 0xBF58476D1CE4E5B9ULL;
    return z ^ (z >> 29);
}

__global__ void k_read(const int4 *a, uint64_t n4, int *out) {
    int acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n4; i += stride) { int4 v = __ldg(a + i); acc += v.x ^ v.y ^ v.z ^ v.w; }
    if (acc == 0x7fffffff) out[0] = acc;
}

// D rows of seeds {a0..a3, b0, b1} in shared memory, as in the scan
template <bool NARROW, int D>
__global__ void k_hash(const uint64_t *seeds, uint64_t n_keys, uint64_t kmask, uint64_t *out) {
    __shared__ uint64_t s[D * 6];
    for (int i = threadIdx.x; i < D * 6; i += blockDim.x) s[i] = seeds[i];
    __syncthreads();
    uint64_t acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_keys; i += stride) {
        const uint64_t x = NARROW ? (uint64_t)(uint32_t)(i * 2654435761u) : canon61((int64_t)mix(i));
#pragma unroll
        for (int r = 0; r < D; ++r) {
            const uint64_t *a = s + r * 6;
            acc += hash_g61_t<NARROW>(a[4], a[5], x) ^ (uint64_t)xi_sign61_t<NARROW>(a, x);
        }
        (void)kmask;
    }
    if (acc == 0x123456789ULL) out[0] = acc;
}

__global__ void k_smem_atom(uint32_t words, uint64_t n, int *out) {
    extern __shared__ int sm[];
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&sm[(uint32_t)mix(i) % words], 1);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

template <int W>
__global__ void k_red(void *base, uint64_t elems, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t j = mix(i) % elems;
        if (W == 4) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"((uint32_t *)base + j) : "memory");
        else asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"((uint64_t *)base + j) : "memory");
    }
}

template <typename F>
static float best_ms(F f, int reps = 5) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 148, dev = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const uint64_t bytes = 12ULL << 30;
    int4 *buf;
    int *o;
    uint64_t *seeds, *osk;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("{\"error\": \"alloc\"}\n"); return 1; }
    cudaMemset(buf, 1, bytes);
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&seeds, 64 * 6 * 8);
    cudaMalloc(&osk, 8);
    {
        uint64_t h[64 * 6];
        uint64_t z = 42;
        for (int i = 0; i < 64 * 6; ++i) { z = z * 6364136223846793005ULL + 1442695040888963407ULL; h[i] = (z >> 3) % SKH_P; }
        cudaMemcpy(seeds, h, sizeof(h), cudaMemcpyHostToDevice);
    }
    const float ms_read = best_ms([&] { k_read<<<sms * 8, 512>>>(buf, bytes / 16, o); });
    const uint64_t nk = 1ULL << 28;
    const float ms_hn = best_ms([&] { k_hash<true, 5><<<sms * 8, 256>>>(seeds, nk, 0, osk); });
    const float ms_hw = best_ms([&] { k_hash<false, 5><<<sms * 8, 256>>>(seeds, nk, 0, osk); });
    const uint64_t na = 1ULL << 30;
    cudaFuncSetAttribute(k_smem_atom, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const float ms_sm = best_ms([&] { k_smem_atom<<<sms * 2, 1024, 5120 * 4>>>(5120, na, o); });
    const uint64_t nr = 1ULL << 28;
    const float ms_r32 = best_ms([&] { k_red<4><<<sms * 8, 512>>>(buf, 1u << 20, nr); });
    const float ms_r64 = best_ms([&] { k_red<8><<<sms * 8, 512>>>(buf, 5ull * 512 * 512, nr); });
    const cudaError_t e = cudaDeviceSynchronize();
    printf("{\"sms\": %d, \"sm_clock_mhz_attr\": %d, \"read_stream_gbs\": %.1f, "
           "\"hash_narrow_pairs_per_s\": %.4g, \"hash_wide_pairs_per_s\": %.4g, "
           "\"atoms_smem_per_s\": %.4g, \"red_l2_u32_hist4mb_per_s\": %.4g, \"red_l2_u64_mat10mb_per_s\": %.4g, "
           "\"status\": \"%s\", \"how\": \"tools/roofs_micro.cu: best of 4 after 1 warm-up, CUDA events; "
           "read: 12 GB LDG.128; hash: d=5 rows of (xi deg-3 + h deg-1) mod 2^61-1 per key (csrc/hash.cuh), 2^28 keys; "
           "atoms: int32 atomicAdd into a 20 KB smem region, random addresses; red: L2 red.add random over the region\"}\n",
           sms, clk / 1000, bytes / ms_read / 1e6, nk * 5.0 / ms_hn * 1e3, nk * 5.0 / ms_hw * 1e3,
           na / ms_sm * 1e3, nr / ms_r32 * 1e3, nr / ms_r64 * 1e3, cudaGetErrorString(e));
    return 0;
}
