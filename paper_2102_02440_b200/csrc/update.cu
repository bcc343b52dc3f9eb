// update.cu — sketch_update_filtered: the fused push-down selection + Fast-AGMS
// build ("sketch building is performed during the selection";
// counter formula PAPER.md:192; partitioned update PAPER.md:221).
//
// One kernel launch scans the table once: predicates are evaluated per tuple,
// the exact survivor count is reduced per warp/CTA, and every surviving tuple
// updates one counter per sketch row of every target sketch.  Counters are
// privatised per CTA in shared memory as int32 where they fit (flushed to the
// int64 HBM sketch at the end, exact because integer addition is associative),
// else updated with int64 L2 atomics.
#include <algorithm>
#include <vector>

#include <stdlib.h>
#include <string.h>

#include "hash.cuh"
#include "internal.cuh"
#include "scan.cuh"

using namespace skb;

namespace {

constexpr int kMaxCols = 16, kMaxPreds = 8, kMaxTargets = 16;

struct UpdPred {
    uint32_t col, kind;
    int64_t lo, hi;
    const int64_t *set;  // device, sorted ascending, unique
    uint32_t n;
};

struct UpdTarget {
    int64_t *counters;
    uint32_t ndim, d, wmask0, wmask1, lw1;  // lw1 = log2(w1)
    uint32_t wmask2, lw2;                   // 3-D tensors: lw2 = log2(w2)
    uint32_t key0, key1, key2;
    int32_t smem_off;     // int32 offset of the privatised copy, -1 = global atomics
    uint32_t cells;       // w0 or w0*w1
    uint32_t seed_off;    // uint64 offset into the shared seed table
};

struct UpdParams {
    const void *col[kMaxCols];
    uint32_t col64;       // bit c set: column c is int64
    uint32_t n_preds, n_targets;
    uint64_t n_rows, rows_per_cta;
    UpdPred pred[kMaxPreds];
    UpdTarget tgt[kMaxTargets];
    const uint64_t *seeds[kMaxTargets];   // device seed tables per target: [ndim][d][6]
    unsigned long long *survivors;
    uint32_t smem_counters;               // number of int32 privatised counters
    uint32_t n_seed_words;                // uint64 words of seeds copied to smem
    uint32_t seeds_byte_off;              // byte offset of the seed table in smem
};

__device__ __forceinline__ int64_t load_val(const UpdParams &p, uint32_t c, uint64_t row) {
    if ((p.col64 >> c) & 1u) return __ldg(reinterpret_cast<const long long *>(p.col[c]) + row);
    return (int64_t)__ldg(reinterpret_cast<const int *>(p.col[c]) + row);
}

__device__ __forceinline__ bool in_set(const int64_t *s, uint32_t n, int64_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        int64_t m = __ldg(reinterpret_cast<const long long *>(s) + mid);
        if (m < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(reinterpret_cast<const long long *>(s) + lo) == v;
}

__global__ void __launch_bounds__(512) k_update_generic(const __grid_constant__ UpdParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *sc = reinterpret_cast<int32_t *>(smem);
    uint64_t *sseed = reinterpret_cast<uint64_t *>(smem + p.seeds_byte_off);
    const uint32_t tid = threadIdx.x, bd = blockDim.x;

    for (uint32_t i = tid; i < p.smem_counters; i += bd) sc[i] = 0;
    for (uint32_t t = 0; t < p.n_targets; ++t) {
        uint32_t words = p.tgt[t].ndim * p.tgt[t].d * 6;
        for (uint32_t i = tid; i < words; i += bd) sseed[p.tgt[t].seed_off + i] = p.seeds[t][i];
    }
    __syncthreads();

    const uint64_t begin = uint64_t(blockIdx.x) * p.rows_per_cta;
    const uint64_t end = min(p.n_rows, begin + p.rows_per_cta);
    uint32_t survivors = 0;
    for (uint64_t row = begin + tid; row < end; row += bd) {
        bool ok = true;
        for (uint32_t q = 0; q < p.n_preds && ok; ++q) {
            const UpdPred &pr = p.pred[q];
            int64_t v = load_val(p, pr.col, row);
            if (pr.kind == SK_PRED_POINT) ok = (v == pr.lo);
            else if (pr.kind == SK_PRED_RANGE) ok = (pr.lo <= v) && (v <= pr.hi);
            else ok = in_set(pr.set, pr.n, v);
        }
        if (!ok) continue;
        ++survivors;
        for (uint32_t t = 0; t < p.n_targets; ++t) {
            const UpdTarget &tg = p.tgt[t];
            const uint64_t *s0 = sseed + tg.seed_off;
            const uint64_t x = canon61(load_val(p, tg.key0, row));
            uint64_t y = 0, z = 0;
            const uint64_t *s1 = s0 + tg.d * 6, *s2 = s1 + tg.d * 6;
            if (tg.ndim >= 2) y = canon61(load_val(p, tg.key1, row));
            if (tg.ndim == 3) z = canon61(load_val(p, tg.key2, row));
            for (uint32_t r = 0; r < tg.d; ++r) {
                const uint64_t *a = s0 + r * 6;
                uint32_t cell = (uint32_t)(hash_g61(a[4], a[5], x) & tg.wmask0);
                int sign = xi_sign61(a, x);
                if (tg.ndim >= 2) {
                    const uint64_t *b = s1 + r * 6;
                    cell = (cell << tg.lw1) | (uint32_t)(hash_g61(b[4], b[5], y) & tg.wmask1);
                    sign *= xi_sign61(b, y);
                }
                if (tg.ndim == 3) {   // cell [h0][h1][h2] += xi0 xi1 xi2
                    const uint64_t *c = s2 + r * 6;
                    cell = (cell << tg.lw2) | (uint32_t)(hash_g61(c[4], c[5], z) & tg.wmask2);
                    sign *= xi_sign61(c, z);
                }
                const uint64_t idx = uint64_t(r) * tg.cells + cell;
                if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + idx], sign);
                else atomicAdd(reinterpret_cast<unsigned long long *>(tg.counters + idx),
                               (unsigned long long)(long long)sign);
            }
        }
    }
    // exact survivor count: warp reduce, one atomic per warp
    uint32_t ws = __reduce_add_sync(0xffffffffu, survivors);
    if ((tid & 31) == 0 && ws && p.survivors) atomicAdd(p.survivors, (unsigned long long)ws);
    __syncthreads();
    // flush the privatised int32 counters into the int64 sketch
    for (uint32_t t = 0; t < p.n_targets; ++t) {
        const UpdTarget &tg = p.tgt[t];
        if (tg.smem_off < 0) continue;
        const uint32_t n = tg.d * tg.cells;
        for (uint32_t i = tid; i < n; i += bd) {
            int32_t v = sc[tg.smem_off + i];
            if (v) atomicAdd(reinterpret_cast<unsigned long long *>(tg.counters + i), (unsigned long long)(long long)v);
        }
    }
}

}  // namespace

static sk_status update_impl(const sk_column *cols, uint32_t n_cols, uint64_t n_rows, const sk_pred *preds,
                             uint32_t n_preds, const sk_target *targets, uint32_t n_targets, int64_t *survivors_dev,
                             const PeerPush *push, void *stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (n_cols > kMaxCols || n_preds > kMaxPreds || n_targets > kMaxTargets)
        return fail(SK_EINVAL, "sketch_update_filtered: too many cols/preds/targets (%u/%u/%u)", n_cols, n_preds, n_targets);
    if ((n_cols && !cols) || (n_preds && !preds) || (n_targets && !targets))
        return fail(SK_EINVAL, "sketch_update_filtered: NULL array");
    UpdParams p;
    memset(&p, 0, sizeof(p));
    p.n_rows = n_rows;
    for (uint32_t c = 0; c < n_cols; ++c) {
        if (cols[c].dtype != SK_INT32 && cols[c].dtype != SK_INT64)
            return fail(SK_EINVAL, "sketch_update_filtered: column %u has bad dtype", c);
        if (!cols[c].data && n_rows) return fail(SK_EINVAL, "sketch_update_filtered: column %u is NULL", c);
        p.col[c] = cols[c].data;
        if (cols[c].dtype == SK_INT64) p.col64 |= 1u << c;
    }
    int device = -1;
    for (uint32_t t = 0; t < n_targets; ++t) {
        const sk_sketch *sk = targets[t].sketch;
        if (!sk) return fail(SK_EINVAL, "sketch_update_filtered: NULL target sketch");
        if (device >= 0 && sk->device != device) return fail(SK_EMISMATCH, "sketch_update_filtered: targets on different devices");
        device = sk->device;
        for (uint32_t q = 0; q < sk->ndim; ++q)
            if (targets[t].key_col[q] >= n_cols) return fail(SK_EINVAL, "sketch_update_filtered: target %u key column out of range", t);
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (device < 0) device = prev;
    SKB_CUDA(cudaSetDevice(device));

    std::vector<void *> tmp;  // stream-ordered temporaries (subset sets)
    auto release = [&]() {
        for (void *q : tmp) cudaFreeAsync(q, stream);
        cudaSetDevice(prev);
    };
    p.n_preds = n_preds;
    for (uint32_t q = 0; q < n_preds; ++q) {
        const sk_pred &pr = preds[q];
        if (pr.col >= n_cols || pr.kind > SK_PRED_SUBSET) {
            release();
            return fail(SK_EINVAL, "sketch_update_filtered: predicate %u invalid", q);
        }
        p.pred[q].col = pr.col;
        p.pred[q].kind = pr.kind;
        p.pred[q].lo = pr.lo;
        p.pred[q].hi = pr.hi;
        if (pr.kind == SK_PRED_SUBSET) {
            if (pr.set_size && !pr.set) { release(); return fail(SK_EINVAL, "sketch_update_filtered: NULL subset"); }
            std::vector<int64_t> s(pr.set, pr.set + pr.set_size);
            std::sort(s.begin(), s.end());
            s.erase(std::unique(s.begin(), s.end()), s.end());
            if (s.size() > 0xFFFFFFFFu) { release(); return fail(SK_EINVAL, "subset too large"); }
            p.pred[q].n = (uint32_t)s.size();
            if (!s.empty()) {
                void *dptr = nullptr;
                cudaError_t e = cudaMallocAsync(&dptr, s.size() * sizeof(int64_t), stream);
                if (e != cudaSuccess) { release(); return cuda_fail(e, "cudaMallocAsync(subset)"); }
                tmp.push_back(dptr);
                e = cudaMemcpyAsync(dptr, s.data(), s.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream);
                if (e != cudaSuccess) { release(); return cuda_fail(e, "cudaMemcpyAsync(subset)"); }
                p.pred[q].set = (const int64_t *)dptr;
            }
        }
    }
    // shared-memory plan: privatise targets in declaration order while they fit
    const uint32_t kSmemBudget = 200 * 1024;
    uint32_t seed_words = 0;
    for (uint32_t t = 0; t < n_targets; ++t) seed_words += targets[t].sketch->ndim * targets[t].sketch->d * 6;
    uint32_t counters_budget = kSmemBudget - seed_words * 8 - 16;
    uint32_t smem_counters = 0;
    p.n_targets = n_targets;
    uint32_t soff = 0;
    for (uint32_t t = 0; t < n_targets; ++t) {
        const sk_sketch *sk = targets[t].sketch;
        UpdTarget &tg = p.tgt[t];
        tg.counters = sk->counters;
        tg.ndim = sk->ndim;
        tg.d = sk->d;
        tg.wmask0 = sk->w[0] - 1;
        tg.wmask1 = sk->ndim >= 2 ? sk->w[1] - 1 : 0;
        tg.lw1 = sk->ndim >= 2 ? (uint32_t)__builtin_ctz(sk->w[1]) : 0;
        tg.wmask2 = sk->ndim == 3 ? sk->w[2] - 1 : 0;
        tg.lw2 = sk->ndim == 3 ? (uint32_t)__builtin_ctz(sk->w[2]) : 0;
        tg.key0 = targets[t].key_col[0];
        tg.key1 = sk->ndim >= 2 ? targets[t].key_col[1] : 0;
        tg.key2 = sk->ndim == 3 ? targets[t].key_col[2] : 0;
        tg.cells = (uint32_t)(sk->n_counters / sk->d);
        tg.seed_off = soff;
        soff += sk->ndim * sk->d * 6;
        p.seeds[t] = sk->seeds_dev;
        uint64_t need = uint64_t(sk->d) * tg.cells;
        if ((smem_counters + need) * 4 <= counters_budget) {
            tg.smem_off = (int32_t)smem_counters;
            smem_counters += (uint32_t)need;
        } else {
            tg.smem_off = -1;
        }
    }
    p.smem_counters = smem_counters;
    p.n_seed_words = seed_words;
    p.seeds_byte_off = ((smem_counters * 4 + 15) / 16) * 16;
    size_t smem = p.seeds_byte_off + size_t(seed_words) * 8;
    p.survivors = reinterpret_cast<unsigned long long *>(survivors_dev);

    if (n_rows == 0) {
        release();
        return push ? peer_push_launch(*push, stream) : SK_OK;
    }
    // optimised persistent scan (scan.cu) unless disabled or outside its envelope
    const char *mode = getenv("COMPASS_SCAN");
    if (!(mode && strcmp(mode, "generic") == 0)) {
        ScanCall sc;
        sc.n_cols = n_cols;
        for (uint32_t c = 0; c < n_cols; ++c) {
            sc.col_ptr[c] = cols[c].data;
            sc.col_bytes[c] = cols[c].dtype == SK_INT64 ? 8 : 4;
            sc.col_domain[c] = cols[c].domain;
        }
        sc.n_rows = n_rows;
        sc.n_preds = n_preds;
        for (uint32_t q = 0; q < n_preds; ++q) {
            sc.pred_col[q] = p.pred[q].col;
            sc.pred_kind[q] = p.pred[q].kind;
            sc.pred_lo[q] = p.pred[q].lo;
            sc.pred_hi[q] = p.pred[q].hi;
            sc.pred_set[q] = p.pred[q].set;
            sc.pred_n[q] = p.pred[q].n;
        }
        sc.n_targets = n_targets;
        for (uint32_t t = 0; t < n_targets; ++t) {
            const sk_sketch *sk = targets[t].sketch;
            sc.tgt_counters[t] = sk->counters;
            sc.tgt_ndim[t] = sk->ndim;
            sc.tgt_d[t] = sk->d;
            sc.tgt_w[t][0] = sk->w[0];
            sc.tgt_key[t][0] = targets[t].key_col[0];
            for (uint32_t q = 1; q < 3; ++q) {
                sc.tgt_w[t][q] = q < sk->ndim ? sk->w[q] : 1;
                sc.tgt_key[t][q] = q < sk->ndim ? targets[t].key_col[q] : 0;
            }
            sc.tgt_seeds[t] = sk->seeds_dev;
            sc.tgt_seeds_host[t] = sk->seeds_host.data();
            sc.tgt_sketch[t] = const_cast<sk_sketch *>(sk);
        }
        sc.survivors = p.survivors;
        if (push) sc.push = *push;
        bool launched = false, pushed = false;
        sk_status st = scan_launch(sc, stream, &launched, &pushed);
        if (st != SK_OK || launched) {
            release();
            if (st == SK_OK && push && !pushed) st = peer_push_launch(*push, stream);
            return st;
        }
    }
    const int block = 512;
    cudaError_t e = cudaFuncSetAttribute(k_update_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { release(); return cuda_fail(e, "cudaFuncSetAttribute"); }
    int sms = 148, occ = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_generic, block, smem);
    occ = std::max(occ, 1);
    uint64_t ctas = uint64_t(sms) * occ;
    ctas = std::min<uint64_t>(ctas, (n_rows + 4095) / 4096);
    ctas = std::max<uint64_t>(ctas, (n_rows + (1ULL << 30) - 1) >> 30);  // int32 privatised counters stay exact
    ctas = std::max<uint64_t>(ctas, 1);
    p.rows_per_cta = (n_rows + ctas - 1) / ctas;
    ctas = (n_rows + p.rows_per_cta - 1) / p.rows_per_cta;
    k_update_generic<<<(unsigned)ctas, block, smem, stream>>>(p);
    count_launch();
    e = cudaGetLastError();
    release();
    if (e != cudaSuccess) return cuda_fail(e, "k_update_generic launch");
    return push ? peer_push_launch(*push, stream) : SK_OK;
}

extern "C" sk_status sketch_update_filtered(const sk_column *cols, uint32_t n_cols, uint64_t n_rows,
                                            const sk_pred *preds, uint32_t n_preds,
                                            const sk_target *targets, uint32_t n_targets,
                                            int64_t *survivors_dev, void *stream) {
    return update_impl(cols, n_cols, n_rows, preds, n_preds, targets, n_targets, survivors_dev, nullptr, stream);
}

// checks a push description and copies it into the kernel-side form
static sk_status push_desc(const sk_peer_push *push, PeerPush *pp) {
    if (!push) return fail(SK_EINVAL, "peer push: NULL description");
    if (push->n_peers == 0 || push->n_peers > kMaxPeers) return fail(SK_EINVAL, "peer push: n_peers %u not in 1..%u", push->n_peers, kMaxPeers);
    if (push->n && (!push->src || !push->dst)) return fail(SK_EINVAL, "peer push: NULL src or dst");
    if ((uintptr_t)push->src & 15) return fail(SK_EINVAL, "peer push: src not 16-byte aligned");
    if (push->owner_mode && (push->rank >= push->n_peers || (push->offset & 1) || push->offset + push->n > push->total))
        return fail(SK_EINVAL, "peer push: owner mode needs rank < n_peers, an even offset and offset + n <= total");
    memset(pp, 0, sizeof(*pp));
    pp->src = push->src;
    pp->n = push->n;
    pp->peers = push->n_peers;
    pp->owner_mode = push->owner_mode ? 1u : 0u;
    pp->rank = push->rank;
    pp->offset = push->offset;
    pp->total = push->total;
    for (uint32_t q = 0; q < push->n_peers; ++q) {
        if (push->n && (!push->dst[q] || ((uintptr_t)push->dst[q] & 15))) return fail(SK_EINVAL, "peer push: dst %u NULL or not 16-byte aligned", q);
        pp->dst[q] = push->dst[q];
    }
    return SK_OK;
}

extern "C" sk_status sketch_update_filtered_push(const sk_column *cols, uint32_t n_cols, uint64_t n_rows,
                                                 const sk_pred *preds, uint32_t n_preds,
                                                 const sk_target *targets, uint32_t n_targets,
                                                 int64_t *survivors_dev, const sk_peer_push *push, void *stream) {
    PeerPush pp;
    sk_status st = push_desc(push, &pp);
    if (st != SK_OK) return st;
    return update_impl(cols, n_cols, n_rows, preds, n_preds, targets, n_targets, survivors_dev, pp.n ? &pp : nullptr, stream);
}

extern "C" sk_status sketch_peer_gather(const sk_peer_push *push, void *stream) {
    if (!push || !push->dst || push->n_peers == 0 || push->n_peers > kMaxPeers || push->rank >= push->n_peers)
        return fail(SK_EINVAL, "peer gather: bad description");
    PeerPush pp;
    memset(&pp, 0, sizeof(pp));
    pp.peers = push->n_peers;
    pp.rank = push->rank;
    pp.total = push->total;
    pp.owner_mode = 1;
    for (uint32_t q = 0; q < push->n_peers; ++q) {
        if (!push->dst[q] || ((uintptr_t)push->dst[q] & 15)) return fail(SK_EINVAL, "peer gather: dst %u NULL or not 16-byte aligned", q);
        pp.dst[q] = push->dst[q];
    }
    return peer_gather_launch(pp, (cudaStream_t)stream);
}

extern "C" sk_status sketch_peer_push(const sk_peer_push *push, void *stream) {
    PeerPush pp;
    sk_status st = push_desc(push, &pp);
    if (st != SK_OK) return st;
    return peer_push_launch(pp, (cudaStream_t)stream);
}
