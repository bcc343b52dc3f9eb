// scan.cu — the optimised fused scan of sketch_update_filtered.
//
// Persistent kernel, one CTA per SM: 20 consumer warps in 4 ring groups of 5, each group
// with its own producer warp (a slow warp holds back only its group's stream; measured
// 3.02 -> 2.75 ms on C4 against one CTA-wide ring).
//   A1  Each producer streams 640-row tiles of the staged columns (predicate
//       columns; key columns too when the table has no predicate) HBM -> smem
//       with cp.async.bulk (TMA bulk copies, UBLKCP) into a 4-8 stage ring
//       guarded by mbarriers (full: tx-count; empty: consumer release).
//   A2  Consumers read 4 rows per lane with 128-bit shared loads and evaluate
//       the conjunction of point / range / subset predicates (one predicate
//       register per row slot; KW variants: all int32 ranges, one key width).
//   A3  One ballot per row slot; survivors' ring positions are popcs of the
//       ballots; only the survivors' key sectors are gathered with predicated
//       cp.async (LDGSTS, .L2::64B) into a per-warp ring, consumed 3 tiles later.
//   A4  Hashes mod 2^61-1 on the integer pipe (hash.cuh; 64x32 lazy Horner for
//       keys < 2^32), or per-sketch lookup tables for matrices over hinted domains.
//   A5  Keys are aggregated per warp with __match_any_sync (leader adds
//       count * xi, exact by linearity).  1-D sketches that fit
//       are privatised as int32 in smem; others get a per-CTA two-choice
//       heavy-hitter table (canonical key -> count) flushed once, misses are
//       buffered per warp and applied 32 at a time with L2 atomics; hinted key
//       domains go through a histogram (hashed once per distinct key).
//   A6  Matrix sketches: per equal-key-pair leader, one cell per
//       row, smem or L2 (trio loop when the hash families equal two privatised
//       1-D sketches').
//   A7  CTA flush: int32 smem counters and heavy-hitter counts -> int64 HBM
//       sketch with red.global.add (order-independent, bit-exact).
#include "scan_kernel.cuh"

namespace skb {
const void *scan_pick_nk1(uint32_t np, int kw, bool fast, int sub, bool t3);   // scan_k1.cu
const void *scan_pick_nk2(uint32_t np, int kw, bool fast, int sub, bool t3);   // scan_k2.cu
const void *scan_pick_nk3(uint32_t np, int kw, bool fast, int sub, bool t3);   // scan_k3.cu
const void *scan_pick_nk4(uint32_t np, int kw, bool fast, int sub, bool t3);   // scan_k4.cu
}  // namespace skb

namespace {

// Histogram-then-sketch epilogue (SURVEY.md §8(d) lever f): every key x with count c in
// [0, domain) adds c * xi_r(x) at bucket h_r(x) of each 1-D sketch on that key column.
// Exact by linearity: identical to adding +-1 once per surviving tuple.
struct EpiTarget {
    int64_t *counters;
    const uint64_t *seeds;   // device [d][6]
    uint32_t d, wmask, cells;
    int32_t smem_off;        // int32 offset of the CTA-private copy, -1 = L2 atomics
};
constexpr int kMaxEpiTargets = 8;
struct EpiParams {
    const uint32_t *hist;
    uint64_t domain;
    uint32_t n_targets, smem_counters;
    EpiTarget tgt[kMaxEpiTargets];
};

__global__ void __launch_bounds__(512) k_hist_epilogue(const __grid_constant__ EpiParams E) {
    extern __shared__ __align__(16) int32_t esc[];
    for (uint32_t i = threadIdx.x; i < E.smem_counters; i += blockDim.x) esc[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < E.domain; x += stride) {
        const uint32_t c = __ldg(E.hist + x);
        if (!c) continue;
        for (uint32_t t = 0; t < E.n_targets; ++t) {
            const EpiTarget &tg = E.tgt[t];
            for (uint32_t r = 0; r < tg.d; ++r) {
                const uint64_t *a = tg.seeds + r * 6;
                // x < domain <= 2^22: the narrow (64x32) hash path
                const uint32_t cell = (uint32_t)(hash_g61_t<true>(__ldg(a + 4), __ldg(a + 5), x) & tg.wmask);
                uint64_t sa[4] = {__ldg(a), __ldg(a + 1), __ldg(a + 2), __ldg(a + 3)};
                const int64_t v = (int64_t)xi_sign61_t<true>(sa, x) * (int64_t)c;
                if (tg.smem_off >= 0) atomicAdd(&esc[tg.smem_off + r * tg.cells + cell], (int32_t)v);
                else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, v);
            }
        }
    }
    __syncthreads();
    for (uint32_t t = 0; t < E.n_targets; ++t) {
        const EpiTarget &tg = E.tgt[t];
        if (tg.smem_off < 0) continue;
        for (uint32_t q = threadIdx.x; q < tg.d * tg.cells; q += blockDim.x) {
            const int32_t v = esc[tg.smem_off + q];
            if (v) red_add_s64(tg.counters + q, (int64_t)v);
        }
    }
}

// hash lookup table of one sketch dimension over keys [0, dom): lut[x * d + r] =
// (h_r(x) & wmask) << 1 | (xi_r(x) < 0)   (H3/H4 for x < 2^32: the narrow path)
__global__ void k_lut_build(const uint64_t *seeds, uint32_t d, uint32_t wmask, uint64_t dom, uint32_t *lut) {
    const uint32_t dp = (d + 3) & ~3u;   // rows padded to a multiple of 4 (128-bit loads)
    const uint64_t total = dom * dp;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t x = e / dp;
        const uint32_t r = (uint32_t)(e % dp);
        if (r >= d) { lut[e] = 0; continue; }
        const uint64_t *a = seeds + r * 6;
        const uint32_t b = (uint32_t)(hash_g61_t<true>(__ldg(a + 4), __ldg(a + 5), x) & wmask);
        uint64_t sa[4] = {__ldg(a), __ldg(a + 1), __ldg(a + 2), __ldg(a + 3)};
        lut[e] = (b << 1) | (xi_sign61_t<true>(sa, x) < 0 ? 1u : 0u);
    }
}

// lookup table of one hash family over keys [0, dom) (see Pend / process_fast): entry x holds
// 8 uint16 fields, field r = ((r * w + (h_r(x) & (w - 1))) << 1) | (xi_r(x) < 0), r < d
// (H3/H4, narrow path: x < 2^32)
__global__ void k_lutx_build(const uint64_t *seeds, uint32_t d, uint32_t w, uint64_t dom, uint4 *lut) {
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < dom; x += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t r = 0; r < d; ++r) {
            const uint64_t *a = seeds + r * 6;
            const uint32_t b = (uint32_t)(hash_g61_t<true>(__ldg(a + 4), __ldg(a + 5), x) & (w - 1));
            uint64_t sa[4] = {__ldg(a), __ldg(a + 1), __ldg(a + 2), __ldg(a + 3)};
            f[r] = ((r * w + b) << 1) | (xi_sign61_t<true>(sa, x) < 0 ? 1u : 0u);
        }
        lut[x] = make_uint4(f[0] | (f[1] << 16), f[2] | (f[3] << 16), f[4] | (f[5] << 16), f[6] | (f[7] << 16));
    }
}

static const void *pick_kernel(uint32_t nk, uint32_t np, int kw, bool fast, int sub, bool t3) {
    switch (nk) {
        case 1: return skb::scan_pick_nk1(np, kw, fast, sub, t3);
        case 2: return skb::scan_pick_nk2(np, kw, fast, sub, t3);
        case 3: return skb::scan_pick_nk3(np, kw, fast, sub, t3);
        default: return skb::scan_pick_nk4(np, kw, fast, sub, t3);
    }
}

}  // namespace

namespace skb {

static sk_status decline(const char *why) {
    if (getenv("COMPASS_SCAN_DEBUG")) fprintf(stderr, "k_scan declined: %s\n", why);
    return SK_OK;
}

// Returns SK_OK and sets *launched if the optimised scan handled the call; leaves
// *launched false (and returns SK_OK) when the call is outside its envelope.
sk_status scan_launch(const ScanCall &c, cudaStream_t stream, bool *launched, bool *pushed) {
    *launched = false;
    *pushed = false;
    if (c.n_cols > kMaxSCols || c.n_preds > 4 || c.n_targets > kMaxSTargets || c.n_rows == 0) return decline("call size");
    SParams P;
    memset(&P, 0, sizeof(P));
    P.n_cols = c.n_cols;
    P.n_rows = c.n_rows;
    for (uint32_t i = 0; i < c.n_cols; ++i) {
        P.col[i].p = c.col_ptr[i];
        P.col[i].bytes = c.col_bytes[i];
        P.col[i].soff = -1;
        if (((uintptr_t)c.col_ptr[i]) & 15) return decline("column alignment");   // bulk copies need 16-byte alignment
    }
    // distinct key columns
    std::vector<uint32_t> keys;
    for (uint32_t t = 0; t < c.n_targets; ++t)
        for (uint32_t q = 0; q < c.tgt_ndim[t]; ++q)
            if (std::find(keys.begin(), keys.end(), c.tgt_key[t][q]) == keys.end()) keys.push_back(c.tgt_key[t][q]);
    if (keys.size() > (size_t)kMaxKeys) return decline("key columns");
    P.n_keys = (uint32_t)keys.size();
    // histogram mode for key columns with a small hinted domain feeding 1-D sketches
    const char *env_hist = getenv("COMPASS_HIST");
    const bool allow_hist = !(env_hist && strcmp(env_hist, "0") == 0) && c.n_rows < (1ULL << 31);
    bool hist_key[kMaxKeys] = {false, false, false, false};
    for (uint32_t k = 0; k < P.n_keys; ++k) {
        bool one_d = false;
        for (uint32_t t = 0; t < c.n_targets; ++t) one_d |= (c.tgt_ndim[t] == 1 && c.tgt_key[t][0] == keys[k]);
        const uint64_t dom = c.col_domain[keys[k]];
        hist_key[k] = allow_hist && one_d && dom > 0 && dom <= (1ULL << 22);
    }
    P.n_preds = c.n_preds;
    for (uint32_t q = 0; q < c.n_preds; ++q) {
        SPred &pr = P.pred[q];
        pr.col = c.pred_col[q];
        pr.set = c.pred_set[q];
        pr.n = c.pred_n[q];
        int64_t lo = c.pred_lo[q], hi = c.pred_kind[q] == SK_PRED_POINT ? c.pred_lo[q] : c.pred_hi[q];
        if (c.pred_kind[q] == SK_PRED_SUBSET) { pr.kind = pr.n ? PR_SET : PR_NONE; continue; }
        if (c.col_bytes[pr.col] == 4) {
            lo = std::max<int64_t>(lo, INT32_MIN);
            hi = std::min<int64_t>(hi, INT32_MAX);
            if (lo > hi) { pr.kind = PR_NONE; continue; }
            pr.kind = PR_R32;
            pr.lo = (int64_t)(uint32_t)(int32_t)lo;
            pr.span = (uint32_t)((int32_t)hi - (int32_t)lo);
        } else {
            if (lo > hi) { pr.kind = PR_NONE; continue; }
            pr.kind = PR_R64;
            pr.lo = lo;
            pr.span = (uint64_t)hi - (uint64_t)lo;
        }
    }
    // ---- lookup-table path (FAST, see process_fast): every key column int32 with a hinted
    //      domain <= 2^22; on each key column one hash family (all its 1-D sketches and matrix
    //      dimensions share d and the seed rows, i.e. the same edge), d <= 8 and d * w <= 2^15 for
    //      the widest 1-D sketch on it (the primary), whose handle caches the table
    bool fast = !(getenv("COMPASS_FAST") && strcmp(getenv("COMPASS_FAST"), "0") == 0) && P.n_keys <= 2 &&
                c.n_preds <= 2 && c.n_rows < (1ULL << 31) && !getenv("COMPASS_SCAN_KW0");
    for (uint32_t q = 0; fast && q < c.n_preds; ++q) fast = P.pred[q].kind == PR_R32;
    int fam_t[kMaxKeys] = {-1, -1, -1, -1};
    for (uint32_t k = 0; fast && k < P.n_keys; ++k) {
        const uint32_t col = keys[k];
        const uint64_t dom = c.col_domain[col];
        fast = c.col_bytes[col] == 4 && dom > 0 && dom <= (1ULL << 22);
        int best = -1;
        for (uint32_t t = 0; fast && t < c.n_targets; ++t)
            if (c.tgt_ndim[t] == 1 && c.tgt_key[t][0] == col && c.tgt_sketch[t] &&
                (best < 0 || c.tgt_w[t][0] > c.tgt_w[best][0]))
                best = (int)t;
        if (!fast || best < 0) { fast = false; break; }
        const uint32_t d = c.tgt_d[best], wmax = c.tgt_w[best][0];
        fast = d <= 8 && d * wmax <= (1u << 15);
        for (uint32_t t = 0; fast && t < c.n_targets; ++t)
            for (uint32_t q = 0; q < c.tgt_ndim[t]; ++q) {
                if (c.tgt_key[t][q] != col) continue;
                if (c.tgt_d[t] != d || c.tgt_w[t][q] > wmax ||
                    memcmp(c.tgt_seeds_host[t] + size_t(q) * d * 6, c.tgt_seeds_host[best], size_t(d) * 6 * 8) != 0)
                    fast = false;
            }
        fam_t[k] = best;
    }
    if (fast) {   // matrix targets of the lookup-table path (both dims on the two key columns)
        P.n_mat = 0;
        for (uint32_t t = 0; t < c.n_targets; ++t)
            if (c.tgt_ndim[t] == 3) fast = false;   // 3-D tensors take the hashing drain
            else if (c.tgt_ndim[t] == 2) {
                if (P.n_mat == 2 || c.tgt_key[t][0] == c.tgt_key[t][1]) fast = false;
                else P.mat_t[P.n_mat++] = t;
            }
    }
    if (fast) {
        int dev_f = 0, sms_f = 148;
        cudaGetDevice(&dev_f);
        cudaDeviceGetAttribute(&sms_f, cudaDevAttrMultiProcessorCount, dev_f);
        for (uint32_t k = 0; k < P.n_keys; ++k) {
            hist_key[k] = false;
            sk_sketch *sk = c.tgt_sketch[fam_t[k]];
            const uint64_t dom = c.col_domain[keys[k]];
            std::lock_guard<std::mutex> lk(sk->lut_mu);
            if (!sk->lutx || sk->lutx_dom < dom) {
                if (sk->lutx) {   // replaced: no reader of the old table may be in flight
                    SKB_CUDA(cudaDeviceSynchronize());
                    cudaFree(sk->lutx);
                    sk->lutx = nullptr;
                }
                SKB_CUDA(cudaMalloc(&sk->lutx, dom * 16));
                k_lutx_build<<<(unsigned)std::min<uint64_t>(uint64_t(sms_f) * 8, (dom + 255) / 256), 256, 0, stream>>>(
                    sk->seeds_dev, sk->d, sk->w[0], dom, sk->lutx);
                SKB_CUDA(cudaGetLastError());
                count_launch();
                sk->lutx_dom = dom;
                if (!sk->lut_ready) SKB_CUDA(cudaEventCreateWithFlags(&sk->lut_ready, cudaEventDisableTiming));
                SKB_CUDA(cudaEventRecord(sk->lut_ready, stream));
            } else if (sk->lut_ready) {
                SKB_CUDA(cudaStreamWaitEvent(stream, sk->lut_ready, 0));   // built on another stream
            }
            P.klut[k] = sk->lutx;
            P.klut_dom[k] = sk->lutx_dom;
            P.kprim[k] = (uint32_t)fam_t[k];
            P.kothers[k] = 0;
            for (uint32_t t = 0; t < c.n_targets; ++t)
                if (c.tgt_ndim[t] == 1 && c.tgt_key[t][0] == keys[k] && t != (uint32_t)fam_t[k]) P.kothers[k] |= 1u << t;
        }
    }
    P.gather = c.n_preds > 0 ? 1u : 0u;
    double sel_est = -1.0;   // expected selectivity of the predicates from the value-domain hints (-1: no hint)
    // predicate path: stages of up to 4 sub-tiles, ~10 KB of predicate columns per stage and
    // group (a single int32 column gets 4 sub-tiles: the per-stage work is amortised over more
    // rows); COMPASS_SUB overrides (experiments)
    {
        uint32_t pbytes = 0;
        std::vector<uint32_t> pc;
        for (uint32_t q = 0; q < c.n_preds; ++q)
            if (std::find(pc.begin(), pc.end(), c.pred_col[q]) == pc.end()) { pc.push_back(c.pred_col[q]); pbytes += c.col_bytes[c.pred_col[q]]; }
        // sub-tiles pay only where most sub-tiles hold no survivor: the expected selectivity
        // from the columns' value-domain hints (uniform reading of each predicate's share of
        // the domain; no hint = 1) must be below 1 %
        double est = 1.0;
        bool hinted = false;
        for (uint32_t q = 0; q < c.n_preds; ++q) {
            const double dom = (double)c.col_domain[c.pred_col[q]];
            if (dom <= 0) continue;
            hinted = true;
            double f = 1.0;
            if (c.pred_kind[q] == SK_PRED_SUBSET) f = c.pred_n[q] / dom;
            else {
                const int64_t hi = c.pred_kind[q] == SK_PRED_POINT ? c.pred_lo[q] : c.pred_hi[q];
                const double lo = std::max<double>(0.0, (double)c.pred_lo[q]), h = std::min<double>(dom - 1, (double)hi);
                f = h >= lo ? (h - lo + 1) / dom : 0.0;
            }
            est *= std::min(1.0, f);
        }
        if (hinted) sel_est = est;
        // 4 sub-tiles (instances exist for the lookup-table path with an int32 predicate
        // column: ~10 KB per stage and group, three stages within 3/5 of the budget), else 1
        uint32_t sub = (P.gather && fast && pbytes == 4 && est < 0.01) ? 4u : 1u;
        if (const char *es = getenv("COMPASS_SUB")) sub = (atoi(es) == 4 && P.gather && fast && pbytes == 4) ? 4u : 1u;
        if (sub == 4 && 3u * kGroups * kTile * pbytes * sub > (227u * 1024u) * 3u / 5u) sub = 1;
        P.sub = sub;
    }
    P.tile_rows = kTile * P.sub;
    P.n_tiles = (c.n_rows + P.tile_rows - 1) / P.tile_rows;
    P.n_full_tiles = (uint32_t)(c.n_rows / P.tile_rows);
    // staged columns: predicate columns, plus key columns when there is no predicate
    uint32_t soff = 0;
    auto stage_col = [&](uint32_t col) {
        if (P.col[col].soff >= 0) return;
        P.col[col].soff = (int32_t)soff;
        soff += P.tile_rows * P.col[col].bytes;
    };
    for (uint32_t q = 0; q < c.n_preds; ++q) stage_col(c.pred_col[q]);
    if (!P.gather) for (uint32_t k : keys) stage_col(k);
    P.stage_bytes = soff;
    // staged columns are read by TMA bulk copies: they must be device memory (a mapped host
    // column — allowed for gathered key columns — sends the call to the grid-stride kernel)
    for (uint32_t ci = 0; ci < c.n_cols; ++ci) {
        if (P.col[ci].soff < 0) continue;
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, c.col_ptr[ci]) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            return decline("staged column not device memory");
        }
    }
    // ---- shared-memory plan (227 KB): barriers | TMA ring (stages x stage) | per-warp key
    //      rings | privatised counters | heavy-hitter tables | seeds.  Tunables via env
    //      (COMPASS_STAGES, COMPASS_HH_LOG2) for experiments only.
    const uint32_t kBudget = 227 * 1024;
    const char *env_st = getenv("COMPASS_STAGES"), *env_hh = getenv("COMPASS_HH_LOG2");
    // two key columns at >= 5 % expected selectivity: 3 stages (the rest of the budget is left
    // to the L1 carve-out; tools/sweep_scan.py, r02 s4d/s4e: C5 T8 0.75 -> 0.70 ms, T9 1.53 ->
    // 1.43, cycle T10 3.52 -> 3.31), else 6 and up to the budget
    const bool few_stages = !env_st && c.n_preds > 0 && P.n_keys >= 2 && sel_est >= 0.05;
    const uint32_t want_stages = env_st ? (uint32_t)atoi(env_st) : (few_stages ? 3u : 6u);
    const uint32_t max_hh = env_hh ? (uint32_t)atoi(env_hh) : 11;
    uint32_t seed_words = 0;
    for (uint32_t t = 0; t < c.n_targets; ++t) seed_words += c.tgt_ndim[t] * c.tgt_d[t] * 6;
    P.seed_words = seed_words;
    const uint32_t seed_bytes = (seed_words * 8 + 15) & ~15u;
    for (uint32_t k = 0; k < P.n_keys; ++k) P.key[k].col = keys[k];
    P.cap = 0;
    P.kb_bytes = 0;
    const uint32_t ring_warps = kWarps;                 // warps owning a survivor-key ring
    const uint32_t min_stages = 3;
    const uint32_t miss_bytes = kWarps * P.n_keys * 32 * 12 + ((kWarps * P.n_keys * 4 + 15) & ~15u) + kMaxKeys * 16 + 16;
    const uint32_t kBarBytes = 2 * kGroups * kMaxStages * 8;
    const uint32_t ring_stage = kGroups * P.stage_bytes;   // one stage of every group's ring
    auto fixed_for = [&](uint32_t kb) {
        return kBarBytes + min_stages * ring_stage + ring_warps * kb + seed_bytes + miss_bytes + kWarps * 128 * 2 + 256;
    };
    if (P.gather) {
        // survivor-key ring per warp: >= one tile slice of survivors (128).  Depth measured on
        // the C5 tables (tools/r02_p48.sh; per-table ms at ring 64 / 128 / 256 / 512): one key
        // column at >= 25 % expected selectivity (C5 T10, 50 %) 1.29 / 1.12 / 1.08 / 0.89 -> 512;
        // two key columns at 2-5 % (T7) -> 128.  With 3 stages (tools/sweep_scan.py, r02 s4d /
        // s4e; ring 64 / 128 / 256): T8 (7.5 %) 1.07 / 0.70 / 0.69 and T9 (19 %, uniform keys)
        // 1.47 / 1.89 / 1.43 -> 256; cycle T10 (50 %) 3.45 / 3.31 / 3.92 -> 128 (512 entries
        // push the 1-D sketches out of shared memory: 2.9 / 4.9 / 12.2 ms).  Only with
        // value-domain hints on the predicates.
        const uint32_t base = P.n_keys == 1 ? 256 : SCAN_CAP2;
        uint32_t cap = base;
        if (sel_est >= 0) {
            if (P.n_keys == 1 && sel_est >= 0.25) cap = 512;
            if (P.n_keys >= 2 && sel_est >= 0.02 && sel_est < 0.05) cap = 128;
            if (P.n_keys >= 2 && sel_est >= 0.05 && sel_est < 0.3) cap = 256;   // T8 7.5 %, T9 19 %
            if (P.n_keys >= 2 && sel_est >= 0.3) cap = 128;                      // cycle T10 50 %
        }
        uint64_t sc1d = 0;
        for (uint32_t t = 0; t < c.n_targets; ++t)
            if (c.tgt_ndim[t] == 1) sc1d += uint64_t(c.tgt_d[t]) * c.tgt_w[t][0] * 4;
        while (cap > base && fixed_for(cap * P.n_keys * 8) + sc1d > kBudget) cap /= 2;
        if (const char *ec = getenv("COMPASS_CAP")) cap = std::max<uint32_t>(64, 1u << (31 - __builtin_clz(std::max(1, atoi(ec)))));
        P.cap = cap;
        P.kb_bytes = P.cap * P.n_keys * 8;
    }
    const uint32_t fixed = fixed_for(P.kb_bytes);
    if (fixed > kBudget) return decline("fixed smem");
    uint32_t avail = kBudget - fixed;
    // privatise targets in declaration order while they fit
    P.n_targets = c.n_targets;
    uint32_t sc_count = 0, seed_off = 0;
    bool key_needs_hh[kMaxKeys] = {false, false, false, false};
    for (uint32_t t = 0; t < c.n_targets; ++t) {
        STarget &tg = P.tgt[t];
        tg.counters = c.tgt_counters[t];
        tg.ndim = c.tgt_ndim[t];
        tg.d = c.tgt_d[t];
        tg.wmask0 = c.tgt_w[t][0] - 1;
        tg.wmask1 = tg.ndim >= 2 ? c.tgt_w[t][1] - 1 : 0;
        tg.lw1 = tg.ndim >= 2 ? (uint32_t)__builtin_ctz(c.tgt_w[t][1]) : 0;
        tg.wmask2 = tg.ndim == 3 ? c.tgt_w[t][2] - 1 : 0;
        tg.lw2 = tg.ndim == 3 ? (uint32_t)__builtin_ctz(c.tgt_w[t][2]) : 0;
        tg.k0 = (uint32_t)(std::find(keys.begin(), keys.end(), c.tgt_key[t][0]) - keys.begin());
        tg.k1 = tg.ndim >= 2 ? (uint32_t)(std::find(keys.begin(), keys.end(), c.tgt_key[t][1]) - keys.begin()) : 0;
        tg.k2 = tg.ndim == 3 ? (uint32_t)(std::find(keys.begin(), keys.end(), c.tgt_key[t][2]) - keys.begin()) : 0;
        const uint64_t cells64 = uint64_t(c.tgt_w[t][0]) * (tg.ndim >= 2 ? c.tgt_w[t][1] : 1) * (tg.ndim == 3 ? c.tgt_w[t][2] : 1);
        if (cells64 * tg.d >= (1ULL << 31)) return decline("tensor cells");   // 32-bit cell arithmetic in the drain
        tg.cells = (uint32_t)cells64;
        tg.seed_off = seed_off;
        seed_off += tg.ndim * tg.d * 6;
        P.seeds[t] = c.tgt_seeds[t];
        const uint64_t need = uint64_t(tg.d) * tg.cells * 4;
        const bool via_hist = tg.ndim == 1 && hist_key[tg.k0];
        if (!via_hist && sc_count * 4 + need <= avail) {
            tg.smem_off = (int32_t)sc_count;
            sc_count += (uint32_t)(need / 4);
        } else {
            tg.smem_off = -1;
        }
        if (tg.ndim >= 2) P.has2d = 1;
        if (tg.ndim == 1) {
            P.key[tg.k0].has1d = 1;
            if (tg.smem_off >= 0) P.key[tg.k0].priv1d |= 1u << t;
            else P.key[tg.k0].glob1d |= 1u << t;
            if (tg.smem_off < 0) { P.key[tg.k0].hasglob = 1; key_needs_hh[tg.k0] = true; }
            if (hist_key[tg.k0] && !(getenv("COMPASS_HISTHH") && strcmp(getenv("COMPASS_HISTHH"), "0") == 0))
                key_needs_hh[tg.k0] = true;
        }
    }
    P.smem_counters = sc_count;
    avail -= (sc_count * 4 + 15) & ~15u;
    P.pairhh_off = -1;
    uint32_t pair_bytes = 0;
    if (fast) {   // the lookup-table path updates non-privatised sketches directly (no heavy hitters)
        for (uint32_t k = 0; k < P.n_keys; ++k) { key_needs_hh[k] = false; P.key[k].hasglob = 0; }
        // a skewed-pair table for the first matrix backed by L2 (2^10 slots, 12 KB)
        for (uint32_t t = 0; t < c.n_targets; ++t)
            if (P.tgt[t].ndim == 2 && P.tgt[t].smem_off < 0 && avail >= (12u << 10) + ring_stage * 2) {
                P.pair_t = t;
                P.pair_log2 = 10;
                pair_bytes = 12u << 10;
                avail -= pair_bytes;
                break;
            }
    }
    // hash lookup tables for matrix dimensions whose key column has a domain hint (the table
    // stays L2-resident: dom * d * 4 bytes <= 64 MB per dimension); built once per sketch
    if (!fast && !(getenv("COMPASS_LUT") && strcmp(getenv("COMPASS_LUT"), "0") == 0)) {
        int dev_l = 0, sms_l = 148;
        cudaGetDevice(&dev_l);
        cudaDeviceGetAttribute(&sms_l, cudaDevAttrMultiProcessorCount, dev_l);
        for (uint32_t t = 0; t < c.n_targets; ++t) {
            STarget &tg = P.tgt[t];
            tg.lut0 = tg.lut1 = tg.lut2 = nullptr;
            if (tg.ndim < 2 || !c.tgt_sketch[t]) continue;
            sk_sketch *sk = c.tgt_sketch[t];
            const int nd = (int)tg.ndim;
            uint64_t dom[3] = {0, 0, 0};
            bool ok = true;
            const uint64_t dp = (sk->d + 3) & ~3u;
            for (int q = 0; q < nd; ++q) {
                dom[q] = c.col_domain[c.tgt_key[t][q]];
                ok &= sk->d <= 8 && dom[q] > 0 && dom[q] <= (1ULL << 31) && dom[q] * dp * 4 <= (64ULL << 20);
            }
            if (!ok) continue;
            std::lock_guard<std::mutex> lk(sk->lut_mu);
            bool built = false;
            for (int q = 0; q < nd; ++q) {
                if (sk->lut[q] && sk->lut_dom[q] >= dom[q]) continue;
                if (sk->lut[q]) {   // a wider table replaces it: no reader of the old one may be in flight
                    SKB_CUDA(cudaDeviceSynchronize());
                    cudaFree(sk->lut[q]);
                    sk->lut[q] = nullptr;
                }
                SKB_CUDA(cudaMalloc(&sk->lut[q], dom[q] * dp * 4));
                k_lut_build<<<(unsigned)std::min<uint64_t>(uint64_t(sms_l) * 8, (dom[q] * dp + 255) / 256), 256, 0, stream>>>(
                    sk->seeds_dev + size_t(q) * sk->d * 6, sk->d, sk->w[q] - 1, dom[q], sk->lut[q]);
                SKB_CUDA(cudaGetLastError());
                count_launch();
                sk->lut_dom[q] = dom[q];
                built = true;
            }
            if (built) {
                if (!sk->lut_ready) SKB_CUDA(cudaEventCreateWithFlags(&sk->lut_ready, cudaEventDisableTiming));
                SKB_CUDA(cudaEventRecord(sk->lut_ready, stream));
            } else if (sk->lut_ready) {
                SKB_CUDA(cudaStreamWaitEvent(stream, sk->lut_ready, 0));   // built on another stream
            }
            tg.lut0 = sk->lut[0];
            tg.lut1 = sk->lut[1];
            tg.lut2 = sk->lut[2];
            tg.lut_dom0 = dom[0];
            tg.lut_dom1 = dom[1];
            tg.lut_dom2 = dom[2];
        }
    }
    // trio detection: matrix M whose dimension-q hash rows equal those of a privatised 1-D
    // sketch on the same key (exact comparison of the coefficient rows; same d)
    P.trio_on = 0;
    for (uint32_t m = 0; !fast && m < c.n_targets && !P.trio_on; ++m) {
        const STarget &M = P.tgt[m];
        if (M.ndim != 2 || M.k0 == M.k1) continue;
        int ab[2] = {-1, -1};
        for (uint32_t q = 0; q < 2; ++q) {
            const uint32_t k = q ? M.k1 : M.k0;
            const uint64_t *rows = c.tgt_seeds_host[m] + size_t(q) * M.d * 6;
            for (uint32_t t = 0; t < c.n_targets && ab[q] < 0; ++t) {
                const STarget &T = P.tgt[t];
                if (T.ndim == 1 && T.k0 == k && T.smem_off >= 0 && T.d == M.d &&
                    memcmp(c.tgt_seeds_host[t], rows, size_t(M.d) * 6 * 8) == 0)
                    ab[q] = (int)t;
            }
        }
        if (ab[0] < 0 || ab[1] < 0) continue;
        P.trio_on = 1;
        P.trio_ka = M.k0;
        P.trio_kb = M.k1;
        P.trio_a = (uint32_t)ab[0];
        P.trio_b = (uint32_t)ab[1];
        P.trio_m = m;
        P.key[M.k0].priv1d &= ~(1u << ab[0]);   // updated in the trio loop, not per key
        P.key[M.k1].priv1d &= ~(1u << ab[1]);
    }
    // ring depth to 4 stages first, then heavy-hitter tables (up to 2^11 slots per key),
    // then further stages up to want_stages
    uint32_t stages = min_stages;
    while (stages < 4 && stages < want_stages && avail >= ring_stage) { ++stages; avail -= ring_stage; }
    uint32_t nhh = 0;
    for (uint32_t k = 0; k < P.n_keys; ++k) nhh += key_needs_hh[k];
    P.hh_log2 = 0;
    for (uint32_t l = max_hh; l >= 8 && nhh; --l)
        if (nhh * (12u << l) <= avail) { P.hh_log2 = l; break; }
    if (P.hh_log2) avail -= nhh * (12u << P.hh_log2);
    while (stages < want_stages && stages < kMaxStages && avail >= ring_stage) { ++stages; avail -= ring_stage; }
    while (stages < kMaxStages && !env_st && !few_stages && avail >= ring_stage && nhh == 0) { ++stages; avail -= ring_stage; }
    P.stages = stages;
    uint32_t off = (kBarBytes + 127) & ~127u;            // full + empty mbarriers per group
    P.off_ring = off;
    off += stages * ring_stage;
    off = (off + 127) & ~127u;
    P.off_kbuf = off;
    off += ring_warps * P.kb_bytes;
    P.off_sc = off;
    off += (sc_count * 4 + 15) & ~15u;
    for (uint32_t k = 0; k < P.n_keys; ++k) {
        P.key[k].hh_off = -1;
        if (key_needs_hh[k] && P.hh_log2) {
            P.key[k].hh_off = (int32_t)off;
            off += 12u << P.hh_log2;
        }
    }
    P.off_rows = (off + 15) & ~15u;
    off = P.off_rows + kWarps * 128 * 2;
    P.off_miss = (off + 15) & ~15u;
    off = P.off_miss + kWarps * P.n_keys * 32 * 12;
    P.off_missn = (off + 15) & ~15u;
    off = P.off_missn + kWarps * P.n_keys * 4;
    if (pair_bytes) {
        P.pairhh_off = (int32_t)((off + 15) & ~15u);
        off = (uint32_t)P.pairhh_off + pair_bytes;
    }
    P.off_hstat = (off + 15) & ~15u;
    off = P.off_hstat + kMaxKeys * 4 * 4;
    P.off_seed = (off + 15) & ~15u;
    off = P.off_seed + seed_bytes;
    if (off > kBudget) return decline("smem plan");
    P.survivors = c.survivors;

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char *es = getenv("COMPASS_SCAN_CTAS")) sms = std::max(1, std::min(sms, atoi(es)));   // experiments
    uint64_t grid = std::min<uint64_t>((uint64_t)sms, (P.n_tiles + kGroups - 1) / kGroups);
    // int32 privatised counts stay exact: rows per CTA < 2^31
    if ((P.n_tiles + grid * kGroups - 1) / (grid * kGroups) * P.tile_rows * kGroups >= (1ULL << 31)) return decline("rows per CTA");
    if (P.n_keys == 0) return decline("no key column");
    std::vector<void *> hists;
    for (uint32_t k = 0; k < P.n_keys; ++k) {
        P.key[k].hist = nullptr;
        P.key[k].domain = 0;
        if (!hist_key[k]) continue;
        void *h = nullptr;
        const uint64_t dom = c.col_domain[keys[k]];
        SKB_CUDA(cudaMallocAsync(&h, dom * 4, stream));
        SKB_CUDA(cudaMemsetAsync(h, 0, dom * 4, stream));
        hists.push_back(h);
        P.key[k].hist = (uint32_t *)h;
        P.key[k].domain = dom;
    }
    // specialisation: all predicates int32 ranges and one key width -> KW, else generic
    int kw = (int)P.col[P.key[0].col].bytes;
    for (uint32_t k = 1; k < P.n_keys; ++k)
        if ((int)P.col[P.key[k].col].bytes != kw) kw = 0;
    for (uint32_t q = 0; q < P.n_preds; ++q)
        if (P.pred[q].kind != PR_R32) kw = 0;
    if (getenv("COMPASS_SCAN_KW0")) kw = 0;   // experiments / parity of the generic variant
    // 3-D tensor targets: the T3 instances (generic KW = 0, hashing drain) carry the tensor code
    bool t3 = false;
    for (uint32_t t = 0; t < c.n_targets; ++t) t3 = t3 || c.tgt_ndim[t] == 3;
    if (t3) kw = 0;
    const void *kern = pick_kernel(P.n_keys, P.n_preds, kw, fast && !t3, (int)P.sub, t3);
    const int threads = kThreads;
    if (getenv("COMPASS_SCAN_DEBUG"))
        fprintf(stderr, "k_scan plan: keys %u preds %u kw %d fast %d stages %u hh_log2 %u cap %u smem %u (ring %u, counters %u)\n",
                P.n_keys, P.n_preds, kw, (int)fast, P.stages, P.hh_log2, P.cap, off, P.stages * kGroups * P.stage_bytes,
                P.smem_counters * 4);
    SKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)off));
    // fused cross-GPU merge: only when no histogram epilogue has to run after the scan (its
    // counts must be in the partial before the push); a cooperative launch guarantees that
    // every CTA is co-resident for the tail's grid barrier
    bool fuse = c.push.peers > 0 && hists.empty();
    void *bar = nullptr;
    if (fuse) {
        P.push = c.push;
        SKB_CUDA(cudaMallocAsync(&bar, 16, stream));
        SKB_CUDA(cudaMemsetAsync(bar, 0, 16, stream));
        P.push_bar = (unsigned int *)bar;
    }
    void *kargs[] = {&P};
    if (fuse) {
        // COMPASS_SCAN_NOCOOP: take the fallback below (tests)
        const cudaError_t e = getenv("COMPASS_SCAN_NOCOOP") ? cudaErrorCooperativeLaunchTooLarge
                              : cudaLaunchCooperativeKernel(kern, dim3((unsigned)grid), dim3(threads), kargs, off, stream);
        if (e == cudaSuccess) {
            *pushed = true;
        } else {   // co-residency not available (e.g. a restricted grid): plain scan, the caller pushes after it
            cudaGetLastError();
            memset(&P.push, 0, sizeof(P.push));
            P.push_bar = nullptr;
            SKB_CUDA(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(threads), kargs, off, stream));
        }
        SKB_CUDA(cudaFreeAsync(bar, stream));
    } else {
        SKB_CUDA(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(threads), kargs, off, stream));
    }
    count_launch();
    // histogram -> sketches, then release the histograms (stream-ordered).  Every 1-D target
    // on a histogram key gets its in-domain counts only here, so all of them must be served:
    // the targets go in chunks of kMaxEpiTargets, one epilogue launch per chunk.
    for (uint32_t k = 0; k < P.n_keys; ++k) {
        if (!P.key[k].hist) continue;
      for (uint32_t t_next = 0; t_next < c.n_targets;) {
        EpiParams E;
        memset(&E, 0, sizeof(E));
        E.hist = P.key[k].hist;
        E.domain = P.key[k].domain;
        uint32_t sc2 = 0;
        uint32_t t = t_next;
        for (; t < c.n_targets && E.n_targets < kMaxEpiTargets; ++t) {
            if (c.tgt_ndim[t] != 1 || c.tgt_key[t][0] != keys[k]) continue;
            EpiTarget &et = E.tgt[E.n_targets++];
            et.counters = c.tgt_counters[t];
            et.seeds = c.tgt_seeds[t];
            et.d = c.tgt_d[t];
            et.wmask = c.tgt_w[t][0] - 1;
            et.cells = c.tgt_w[t][0];
            const uint32_t need = et.d * et.cells;
            if ((sc2 + need) * 4 <= 200 * 1024) { et.smem_off = (int32_t)sc2; sc2 += need; }
            else et.smem_off = -1;
        }
        t_next = t;
        if (!E.n_targets) break;
        E.smem_counters = sc2;
        const size_t esm = size_t(sc2) * 4;
        SKB_CUDA(cudaFuncSetAttribute(k_hist_epilogue, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm));
        const unsigned eg = (unsigned)std::min<uint64_t>(uint64_t(sms), (E.domain + 511) / 512);
        k_hist_epilogue<<<std::max(1u, eg), 512, esm, stream>>>(E);
        SKB_CUDA(cudaGetLastError());
        count_launch();
      }
    }
    for (void *h : hists) cudaFreeAsync(h, stream);
    *launched = true;
    return SK_OK;
}

}  // namespace skb
