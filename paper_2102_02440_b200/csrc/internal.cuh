// internal.cuh — private declarations of libcompass_b200 (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "compass_b200.h"

// Mersenne prime of the hash family, p = 2^61 - 1.
#define SKP_MERSENNE61 0x1FFFFFFFFFFFFFFFULL

struct sk_sketch {
    uint32_t d = 0, ndim = 0, w[3] = {0, 0, 0};
    uint64_t master = 0;
    std::string edge[3];
    int device = 0;
    int64_t *counters = nullptr;
    bool owned = false;
    uint64_t n_counters = 0;
    // per dimension q, per row r: {a0, a1, a2, a3, b0, b1} (H2), on device and host
    uint64_t *seeds_dev = nullptr;
    std::vector<uint64_t> seeds_host;
    // per dimension q: hash lookup table over a hinted key domain [0, lut_dom[q]):
    // lut[q][x * dp + r] = (h_r(x) & (w_q - 1)) << 1 | (xi_r(x) < 0), dp = d rounded up to a
    // multiple of 4 (d <= 8); built on first use
    // (the seeds never change), freed with the sketch
    uint32_t *lut[3] = {nullptr, nullptr, nullptr};
    uint64_t lut_dom[3] = {0, 0, 0};
    // 1-D sketches: lookup table over a hinted key domain [0, lutx_dom) for the scan's
    // lookup-table path (d <= 8, d * w <= 2^15): lutx[x] holds 8 uint16 fields, field r =
    // ((r * w + (h_r(x) & (w - 1))) << 1) | (xi_r(x) < 0) for r < d (H3/H4), i.e. the
    // counter index inside the sketch and the sign
    uint4 *lutx = nullptr;
    uint64_t lutx_dom = 0;
    // the tables are built on the first caller's stream: later calls on any stream wait on
    // this event (recorded after the build); the mutex guards the cache fields
    cudaEvent_t lut_ready = nullptr;
    std::mutex lut_mu;
};

namespace skb {

sk_status fail(sk_status st, const char *fmt, ...);
sk_status cuda_fail(cudaError_t e, const char *what);
void clear_error();

// host seed derivation (H2): coefficient c(master, edge, row, role, idx) mod p
uint64_t seed_coef(uint64_t master, const std::string &edge, uint32_t row, uint32_t role, uint32_t idx);

bool same_desc(const sk_sketch *a, const sk_sketch *b);

// keep the device's default memory pool from releasing memory at every sync
void ensure_pool(int device);

// count one kernel launch issued by the library (sk_kernel_launches)
void count_launch(uint64_t n = 1);

// estimate engine entry used by estimate_join / estimate_subplans / plan_greedy.
// rows_exact (optional): per-row exact decimal strings.
sk_status estimate_mask(const sk_graph *g, uint64_t mask, double *est, double *row_est,
                        std::vector<std::string> *rows_exact, cudaStream_t stream);

}  // namespace skb

#define SKB_CUDA(call)                                           \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) return skb::cuda_fail(e_, #call); \
    } while (0)

#define SKB_CUDA_CHECK(what)                                     \
    do {                                                         \
        cudaError_t e_ = cudaGetLastError();                     \
        if (e_ != cudaSuccess) return skb::cuda_fail(e_, what);  \
    } while (0)
