// c4_floor_micro.cu — memory-system floor of the C4 access pattern, no hashing:
// stream 3 int32 predicate columns (uniform [0,1000), keep v < 368 on each: 4.98%),
// and for survivors load 0, 1 or 2 int64 key columns (sector gathers), XOR-reduced.
// Also: the same with the key columns streamed in full.  Grid-stride LDG.128, full occupancy.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/c4_floor_micro tools/c4_floor_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fill(int *p, uint64_t n, uint64_t seed) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ULL;
        z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ULL; z ^= z >> 29;
        p[i] = (int)((z >> 20) % 1000);
    }
}

template <int NKEY, int HINT>
__global__ void __launch_bounds__(512) k_floor(const int4 *a, const int4 *b, const int4 *c, const long long *k1,
                                                const long long *k2, uint64_t n4, unsigned long long *out) {
    unsigned long long acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const int4 x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i);
        const int m[4] = {x.x < 368 && y.x < 368 && z.x < 368, x.y < 368 && y.y < 368 && z.y < 368,
                          x.z < 368 && y.z < 368 && z.z < 368, x.w < 368 && y.w < 368 && z.w < 368};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!m[j]) continue;
            acc += 1;
            long long v;
            if (NKEY >= 1) {
                if (HINT) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(k1 + i * 4 + j));
                else v = __ldg(k1 + i * 4 + j);
                acc ^= v;
            }
            if (NKEY >= 2) {
                if (HINT) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(k2 + i * 4 + j));
                else v = __ldg(k2 + i * 4 + j);
                acc ^= v;
            }
        }
    }
    if (acc == 0x12345) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_full(const int4 *a, const int4 *b, const int4 *c, const longlong2 *k1,
                                               const longlong2 *k2, uint64_t n4, unsigned long long *out) {
    unsigned long long acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const int4 x = __ldg(a + i), y = __ldg(b + i), z = __ldg(c + i);
        const longlong2 p = __ldg(k1 + 2 * i), q = __ldg(k1 + 2 * i + 1), r = __ldg(k2 + 2 * i), s = __ldg(k2 + 2 * i + 1);
        acc += (x.x < 368) + y.y + z.z + p.x + q.y + r.x + s.y;
    }
    if (acc == 0x12345) out[0] = acc;
}

int main() {
    const uint64_t n = 1000000000ULL, n4 = n / 4;
    int *p[3];
    long long *k[2];
    for (int i = 0; i < 3; ++i) { cudaMalloc(&p[i], n * 4); k_fill<<<148 * 8, 512>>>(p[i], n, 1000003ULL * (i + 1)); }
    for (int i = 0; i < 2; ++i) { cudaMalloc(&k[i], n * 8); cudaMemset(k[i], 1, n * 8); }
    unsigned long long *o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep && ms < best) best = ms;
        }
        printf("%-34s %8.3f ms\n", name, best);
    };
    const int4 *a = (const int4 *)p[0], *b = (const int4 *)p[1], *c = (const int4 *)p[2];
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
        printf("grid %d x 512\n", g);
        run("stream 3 preds", [&] { k_floor<0, 0><<<g, 512>>>(a, b, c, k[0], k[1], n4, o); });
        run("+ gather 1 key (ldg)", [&] { k_floor<1, 0><<<g, 512>>>(a, b, c, k[0], k[1], n4, o); });
        run("+ gather 2 keys (ldg)", [&] { k_floor<2, 0><<<g, 512>>>(a, b, c, k[0], k[1], n4, o); });
        run("+ gather 2 keys (L2::64B)", [&] { k_floor<2, 1><<<g, 512>>>(a, b, c, k[0], k[1], n4, o); });
        run("stream all 5 columns (28 GB)", [&] { k_full<<<g, 512>>>(a, b, c, (const longlong2 *)k[0], (const longlong2 *)k[1], n4, o); });
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
