// api.cu — sketch lifecycle, seeds, merge and error reporting of libcompass_b200.
//
// Seeds follow SURVEY.md §8(c) H2 (the paper leaves the hash family open,
// PAPER.md:152): coefficient = splitmix64(master ^ splitmix64(fnv1a64(edge) ^
// splitmix64(row<<8 | role<<4 | idx))) mod (2^61-1); xi uses a0..a3 (role 0),
// h uses b0, b1 (role 1).  Both endpoints of an edge get identical seeds
// (PAPER.md:148), two edges on one column get different seeds.
#include <stdarg.h>

#include <atomic>
#include <stdio.h>
#include <string.h>

#include "internal.cuh"

namespace skb {

static thread_local std::string g_err = "no error";

sk_status fail(sk_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

sk_status cuda_fail(cudaError_t e, const char *what) {
    return fail(SK_ECUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
}

void clear_error() { g_err = "no error"; }

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t str_hash(const std::string &s) {
    uint64_t h = 0xCBF29CE484222325ULL;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001B3ULL;
    }
    return h;
}

uint64_t seed_coef(uint64_t master, const std::string &edge, uint32_t row, uint32_t role, uint32_t idx) {
    uint64_t lane = mix64((uint64_t(row) << 8) | (uint64_t(role) << 4) | uint64_t(idx));
    uint64_t v = mix64(master ^ mix64(str_hash(edge) ^ lane));
    return v % SKP_MERSENNE61;
}

// Stream-ordered temporaries (cudaMallocAsync) come from the device's default pool; keep
// freed blocks in the pool instead of releasing them to the driver at every synchronisation.
void ensure_pool(int device) {
    static std::atomic<uint64_t> done{0};
    if (device < 0 || device >= 64 || ((done.load() >> device) & 1ULL)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ULL;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.fetch_or(1ULL << device);
}

bool same_desc(const sk_sketch *a, const sk_sketch *b) {
    if (a->d != b->d || a->ndim != b->ndim || a->master != b->master) return false;
    for (uint32_t q = 0; q < a->ndim; ++q)
        if (a->w[q] != b->w[q] || a->edge[q] != b->edge[q]) return false;
    return true;
}

}  // namespace skb

using namespace skb;

static bool is_pow2(uint32_t v) { return v >= 2 && (v & (v - 1)) == 0; }

extern "C" const char *sk_last_error(void) { return g_err.c_str(); }

extern "C" const char *sk_version(void) { return "compass_b200 0.1 (sm_100a)"; }

extern "C" uint64_t sk_kernel_launches(void) { return g_launches.load(); }

extern "C" sk_status sketch_create(const sk_desc *desc, int device, int64_t *counters_dev, sk_sketch **out) {
    if (!desc || !out) return fail(SK_EINVAL, "sketch_create: NULL argument");
    *out = nullptr;
    if (desc->d < 1 || desc->d > 63 || (desc->d % 2) == 0)
        return fail(SK_EINVAL, "sketch_create: d=%u must be odd in [1,63]", desc->d);
    if (desc->ndim < 1 || desc->ndim > 3) return fail(SK_EINVAL, "sketch_create: ndim must be 1, 2 or 3");
    uint64_t cells = 1;
    for (uint32_t q = 0; q < desc->ndim; ++q) {
        if (!is_pow2(desc->w[q]) || desc->w[q] > (1u << 24))
            return fail(SK_EINVAL, "sketch_create: w[%u]=%u must be a power of two in [2, 2^24]", q, desc->w[q]);
        if (!desc->edge_id[q] || !desc->edge_id[q][0]) return fail(SK_EINVAL, "sketch_create: empty edge id");
        cells *= desc->w[q];
    }
    for (uint32_t q = 1; q < desc->ndim; ++q)
        if (strcmp(desc->edge_id[q - 1], desc->edge_id[q]) >= 0)
            return fail(SK_EINVAL, "sketch_create: dims must be in canonical edge order (edge_id[q-1] < edge_id[q])");
    if (cells * desc->d > (1ULL << 31)) return fail(SK_EINVAL, "sketch_create: sketch too large");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SK_ECUDA, "sketch_create: no CUDA device");
    if (device < 0 || device >= ndev) return fail(SK_EINVAL, "sketch_create: bad device %d", device);

    sk_sketch *sk = new sk_sketch();
    sk->d = desc->d;
    sk->ndim = desc->ndim;
    sk->master = desc->master_seed;
    for (uint32_t q = 0; q < desc->ndim; ++q) {
        sk->w[q] = desc->w[q];
        sk->edge[q] = desc->edge_id[q];
    }
    sk->device = device;
    sk->n_counters = cells * desc->d;
    ensure_pool(device);
    sk->seeds_host.resize(size_t(sk->ndim) * sk->d * 6);
    for (uint32_t q = 0; q < sk->ndim; ++q)
        for (uint32_t r = 0; r < sk->d; ++r) {
            uint64_t *s = &sk->seeds_host[(size_t(q) * sk->d + r) * 6];
            for (uint32_t i = 0; i < 4; ++i) s[i] = seed_coef(sk->master, sk->edge[q], r, 0, i);
            for (uint32_t i = 0; i < 2; ++i) s[4 + i] = seed_coef(sk->master, sk->edge[q], r, 1, i);
        }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&sk->seeds_dev, sk->seeds_host.size() * sizeof(uint64_t));
    if (e == cudaSuccess)
        e = cudaMemcpy(sk->seeds_dev, sk->seeds_host.data(), sk->seeds_host.size() * sizeof(uint64_t),
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        if (counters_dev) {
            sk->counters = counters_dev;
        } else {
            e = cudaMalloc(&sk->counters, sk->n_counters * sizeof(int64_t));
            if (e == cudaSuccess) {
                sk->owned = true;
                e = cudaMemset(sk->counters, 0, sk->n_counters * sizeof(int64_t));
            }
        }
    }
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        sketch_destroy(sk);
        return cuda_fail(e, "sketch_create");
    }
    *out = sk;
    return SK_OK;
}

extern "C" sk_status sketch_destroy(sk_sketch *sk) {
    if (!sk) return SK_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(sk->device);
    cudaDeviceSynchronize();
    if (sk->owned && sk->counters) cudaFree(sk->counters);
    if (sk->seeds_dev) cudaFree(sk->seeds_dev);
    for (int q = 0; q < 3; ++q)
        if (sk->lut[q]) cudaFree(sk->lut[q]);
    if (sk->lutx) cudaFree(sk->lutx);
    if (sk->lut_ready) cudaEventDestroy(sk->lut_ready);
    cudaSetDevice(prev);
    delete sk;
    return SK_OK;
}

extern "C" sk_status sketch_counters(const sk_sketch *sk, int64_t **counters_dev, uint64_t *n_counters) {
    if (!sk) return fail(SK_EINVAL, "sketch_counters: NULL sketch");
    if (counters_dev) *counters_dev = sk->counters;
    if (n_counters) *n_counters = sk->n_counters;
    return SK_OK;
}

extern "C" sk_status sketch_zero(sk_sketch *sk, void *stream) {
    if (!sk) return fail(SK_EINVAL, "sketch_zero: NULL sketch");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(sk->device);
    cudaError_t e = cudaMemsetAsync(sk->counters, 0, sk->n_counters * sizeof(int64_t), (cudaStream_t)stream);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "sketch_zero");
    return SK_OK;
}

// dst += src: 128-bit vectorised elementwise add over the int64 counters.
__global__ void k_merge_add(int64_t *__restrict__ dst, const int64_t *__restrict__ src, uint64_t n) {
    uint64_t n2 = n / 2;
    uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) {
        longlong2 a = reinterpret_cast<longlong2 *>(dst)[i];
        longlong2 b = reinterpret_cast<const longlong2 *>(src)[i];
        a.x += b.x;
        a.y += b.y;
        reinterpret_cast<longlong2 *>(dst)[i] = a;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[n - 1] += src[n - 1];
}

// int32 wire format of the cross-GPU merge (SURVEY.md §8(e) lever i): exact while every
// partial and merged counter lies in int32, i.e. every table has < 2^31 rows (|counter| <=
// survivors).  A value outside int32 sets *overflow (device flag, never cleared here).
__global__ void k_wire_pack(const int64_t *src, int32_t *dst, uint64_t n, unsigned int *overflow) {
    bool bad = false;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const int64_t v = src[i];
        bad |= v != (int64_t)(int32_t)v;
        dst[i] = (int32_t)v;
    }
    if (bad && overflow) atomicOr(overflow, 1u);
}
__global__ void k_wire_unpack(const int32_t *src, int64_t *dst, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] = (int64_t)src[i];
}

extern "C" sk_status sketch_wire_pack(const int64_t *counters_dev, int32_t *wire_dev, uint64_t n, unsigned int *overflow_dev,
                                      void *stream) {
    if (n && (!counters_dev || !wire_dev)) return fail(SK_EINVAL, "sketch_wire_pack: NULL buffer");
    if (!n) return SK_OK;
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
    k_wire_pack<<<blocks, 256, 0, (cudaStream_t)stream>>>(counters_dev, wire_dev, n, overflow_dev);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SK_OK : cuda_fail(e, "sketch_wire_pack launch");
}

extern "C" sk_status sketch_wire_unpack(const int32_t *wire_dev, int64_t *counters_dev, uint64_t n, void *stream) {
    if (n && (!counters_dev || !wire_dev)) return fail(SK_EINVAL, "sketch_wire_unpack: NULL buffer");
    if (!n) return SK_OK;
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
    k_wire_unpack<<<blocks, 256, 0, (cudaStream_t)stream>>>(wire_dev, counters_dev, n);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SK_OK : cuda_fail(e, "sketch_wire_unpack launch");
}

extern "C" sk_status sketch_merge(sk_sketch *dst, const sk_sketch *src, void *stream) {
    if (!dst || !src) return fail(SK_EINVAL, "sketch_merge: NULL sketch");
    if (!same_desc(dst, src)) return fail(SK_EMISMATCH, "sketch_merge: descriptors differ (d, ndim, w, seed or edge ids)");
    if (dst->device != src->device) return fail(SK_EMISMATCH, "sketch_merge: sketches on different devices");
    if (dst == src) return fail(SK_EINVAL, "sketch_merge: dst == src");
    if (((uintptr_t)dst->counters | (uintptr_t)src->counters) & 15)
        return fail(SK_EINVAL, "sketch_merge: counters must be 16-byte aligned");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dst->device);
    int blocks = (int)std::min<uint64_t>((dst->n_counters / 2 + 255) / 256 + 1, 148 * 8);
    k_merge_add<<<blocks, 256, 0, (cudaStream_t)stream>>>(dst->counters, src->counters, dst->n_counters);
    count_launch();
    cudaError_t e = cudaGetLastError();
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "sketch_merge launch");
    return SK_OK;
}
