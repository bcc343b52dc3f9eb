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
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <mutex>
#include <vector>

#include "hash.cuh"
#include "internal.cuh"
#include "scan.cuh"

using namespace skb;

namespace {

#ifndef SCAN_WAIT_HINT
#define SCAN_WAIT_HINT 1
#endif
#ifndef SCAN_CAP2
#define SCAN_CAP2 64
#endif
#ifndef SCAN_WARPS
#define SCAN_WARPS 20
#endif
#ifndef SCAN_GROUPS
#define SCAN_GROUPS 4
#endif
constexpr int kWarps = SCAN_WARPS;           // consumer warps per CTA
constexpr int kGroups = SCAN_GROUPS;         // independent ring groups per CTA (one producer warp each)
constexpr int kGW = kWarps / kGroups;        // consumer warps per group
constexpr int kTile = kGW * 128;             // rows per group tile (one ring stage)
static_assert(kWarps % kGroups == 0, "warps must split evenly into ring groups");

constexpr int kConsumers = kWarps * 32;
constexpr int kThreads = kConsumers + 32 * kGroups;
constexpr int kMaxStages = 8;
constexpr int kMaxSCols = 8, kMaxSPreds = 8, kMaxKeys = 4, kMaxSTargets = 16;
constexpr uint64_t kEmpty = ~0ULL;   // canonical keys are < 2^61: never equal

struct SCol {
    const void *p;
    uint32_t bytes;       // 4 or 8
    int32_t soff;         // byte offset inside a stage, -1 = not staged
};
enum { PR_R32 = 0, PR_R64 = 1, PR_SET = 2, PR_NONE = 3 };
struct SPred {
    uint32_t col, kind;   // PR_R32: (uint32)(v - lo32) <= span32; PR_R64: (uint64)(v - lo) <= span; PR_NONE: no row
    int64_t lo;           // POINT c is RANGE [c, c]
    uint64_t span;
    const int64_t *set;
    uint32_t n;
};
struct SKey {
    uint32_t col;
    int32_t hh_off;       // byte offset of this key's heavy-hitter table, -1 = none
    uint32_t has1d;       // some 1-D target hashes this key
    uint32_t hasglob;     // some non-privatised 1-D target hashes this key
    uint32_t *hist;       // histogram mode: per-key counts over [0, domain), else null
    uint64_t domain;
    uint32_t priv1d;      // bit t: 1-D target t on this key, privatised in smem
    uint32_t glob1d;      // bit t: 1-D target t on this key, updated in HBM/L2
};
struct STarget {
    int64_t *counters;
    uint32_t ndim, d, wmask0, wmask1, lw1;
    uint32_t k0, k1;      // indices into keys[]
    int32_t smem_off;     // int32 offset of privatised copy, -1 = global
    uint32_t cells;
    uint32_t seed_off;
    const uint32_t *lut0, *lut1;   // matrices: per-dimension hash lookup tables (or null)
    uint64_t lut_dom0, lut_dom1;
};
struct SParams {
    SCol col[kMaxSCols];
    SPred pred[kMaxSPreds];
    SKey key[kMaxKeys];
    STarget tgt[kMaxSTargets];
    const uint64_t *seeds[kMaxSTargets];
    uint32_t n_cols, n_preds, n_keys, n_targets;
    uint64_t n_rows, n_tiles;
    uint32_t stage_bytes;
    uint32_t stages;      // ring depth (<= kMaxStages)
    uint32_t gather;      // 1: survivors' keys gathered, 0: keys staged (no predicate)
    uint32_t cap;         // entries of each warp's survivor-key ring (power of two)
    uint32_t kb_bytes;    // bytes of one warp's ring
    uint32_t hh_log2;     // heavy-hitter slots per key = 1 << hh_log2
    // smem layout (byte offsets)
    uint32_t off_ring, off_kbuf, off_hh, off_sc, off_seed;
    uint32_t smem_counters, seed_words;
    uint32_t has2d;       // some target is a matrix
    // trio: a matrix M on key columns (ka, kb) whose two hash families equal those of the
    // privatised 1-D sketches A on ka and B on kb (same edges, same d).  One row loop hashes
    // each survivor's two keys once and updates A, B and M (the matrix reuses the 1-D hash
    // values).
    uint32_t trio_on, trio_ka, trio_kb, trio_a, trio_b, trio_m;
    uint32_t off_miss, off_missn;   // per-warp miss buffers (x, count) and fill counts
    uint32_t off_hstat;             // per key: heavy-hitter probes, hits, disabled flag (histogram keys)
    uint32_t off_rows;              // per-warp survivor row-offset list (128 x uint16)
    uint32_t tile_rows;             // rows per ring stage
    uint32_t n_full_tiles;          // tiles with tile_rows rows (staged by TMA)
    unsigned long long *survivors;
};

// ------------------------------------------------------------------ PTX helpers
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
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity), "r"(0x989680u) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
#if SCAN_WAIT_HINT
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(bar), "r"(parity), "r"(0x989680u) : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
#endif
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// every committed group has landed (cp.async issued since the last commit are not covered)
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// commits the current (possibly partial) group too: every cp.async issued so far has landed
__device__ __forceinline__ void cp_commit_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
#ifndef SCAN_LAG
#define SCAN_LAG 3
#endif
constexpr int kLag = SCAN_LAG;   // a tile's gathered keys are consumed kLag tiles later
__device__ __forceinline__ void cp_wait_lag() { asm volatile("cp.async.wait_group %0;" ::"n"(kLag) : "memory"); }
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }
__device__ __forceinline__ void red_add_u32(uint32_t *p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_s64(int64_t *p, int64_t v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ bool in_set(const int64_t *s, uint32_t n, int64_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(reinterpret_cast<const long long *>(s) + mid) < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(reinterpret_cast<const long long *>(s) + lo) == v;
}

// ------------------------------------------------------------------ heavy-hitter table
// Two-choice table of 2^log2s slots (canonical key -> int32 count): a key lives in slot
// s1(x) or s2(x); a probe is one 64-bit shared load and compare per choice, so a hit on
// the first choice (every hot key: they arrive first) costs a handful of instructions.
// Slots are never freed, so a key found in s2 cannot also sit in s1.  Two warps may
// still insert one key twice in a race; both counts are flushed, which is exact by
// linearity.
__device__ __forceinline__ uint64_t lds_v64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ bool hh_add(unsigned char *tab, uint32_t log2s, uint64_t x, int cnt) {
    // shared-window addresses and shared-space atomics (no generic-address conversion)
    const uint32_t ka = smem_u32(tab), ca = ka + (8u << log2s);
    const uint64_t h = x * 0x9E3779B97F4A7C15ULL;
    const uint32_t mask = (1u << log2s) - 1u;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const uint32_t sl = (uint32_t)(h >> (c ? 24 : 44)) & mask;
        uint64_t k = lds_v64(ka + sl * 8);
        if (k == kEmpty)
            asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(k) : "r"(ka + sl * 8), "l"(kEmpty), "l"(x) : "memory");
        if (k == x || k == kEmpty) {
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(ca + sl * 4), "r"(cnt) : "memory");
            return true;
        }
    }
    return false;
}

// ------------------------------------------------------------------ sketch updates
// 1-D target t: row r gets cnt * xi_r(x) at bucket h_r(x)
template <bool N>
__device__ __forceinline__ void update_1d_t(const STarget &tg, const uint64_t *seed, int32_t *sc, uint64_t x, int cnt) {
    for (uint32_t r = 0; r < tg.d; ++r) {
        const uint64_t *a = seed + r * 6;
        const uint32_t cell = (uint32_t)(hash_g61_t<N>(a[4], a[5], x) & tg.wmask0);
        const int v = xi_sign61_t<N>(a, x) * cnt;
        if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + r * tg.cells + cell], v);
        else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, (int64_t)v);
    }
}
__device__ __forceinline__ void update_1d(const STarget &tg, const uint64_t *seed, int32_t *sc, uint64_t x, int cnt) {
    if (x < (1ULL << 32)) update_1d_t<true>(tg, seed, sc, x, cnt);
    else update_1d_t<false>(tg, seed, sc, x, cnt);
}

template <bool N>
__device__ __forceinline__ void update_2d_t(const STarget &tg, const uint64_t *seed, int32_t *sc, uint64_t x, uint64_t y,
                                            int cnt) {
    const uint64_t *s1 = seed + tg.d * 6;
    for (uint32_t r = 0; r < tg.d; ++r) {
        const uint64_t *a = seed + r * 6, *b = s1 + r * 6;
        const uint32_t cell = ((uint32_t)(hash_g61_t<N>(a[4], a[5], x) & tg.wmask0) << tg.lw1) |
                              (uint32_t)(hash_g61_t<N>(b[4], b[5], y) & tg.wmask1);
        const int v = xi_sign61_t<N>(a, x) * xi_sign61_t<N>(b, y) * cnt;
        if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + r * tg.cells + cell], v);
        else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, (int64_t)v);
    }
}
__device__ __forceinline__ void update_2d(const STarget &tg, const uint64_t *seed, int32_t *sc, uint64_t x, uint64_t y,
                                          int cnt) {
    if (tg.lut0 && x < tg.lut_dom0 && y < tg.lut_dom1) {
        // hinted key domains: (bucket, sign) per row from the lookup tables (the same values
        // the hash polynomials give; built once per sketch by k_lut_build)
        // rows padded to a multiple of 4: the entries of both keys arrive in 128-bit loads,
        // all issued before the first use
        const uint32_t dp = (tg.d + 3) & ~3u;
        const uint4 *la = reinterpret_cast<const uint4 *>(tg.lut0 + x * dp), *lb = reinterpret_cast<const uint4 *>(tg.lut1 + y * dp);
        uint4 va[2], vb[2];
        va[0] = __ldg(la); vb[0] = __ldg(lb);
        if (dp > 4) { va[1] = __ldg(la + 1); vb[1] = __ldg(lb + 1); }
        for (uint32_t r = 0; r < tg.d && r < 8; ++r) {
            const uint4 &qa = va[r >> 2], &qb = vb[r >> 2];
            const uint32_t ea = (r & 3) == 0 ? qa.x : (r & 3) == 1 ? qa.y : (r & 3) == 2 ? qa.z : qa.w;
            const uint32_t eb = (r & 3) == 0 ? qb.x : (r & 3) == 1 ? qb.y : (r & 3) == 2 ? qb.z : qb.w;
            const uint32_t cell = ((ea >> 1) << tg.lw1) | (eb >> 1);
            const int v = ((ea ^ eb) & 1u) ? -cnt : cnt;
            if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + r * tg.cells + cell], v);
            else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, (int64_t)v);
        }
        return;
    }
    if ((x | y) < (1ULL << 32)) update_2d_t<true>(tg, seed, sc, x, y, cnt);
    else update_2d_t<false>(tg, seed, sc, x, y, cnt);
}

// x[idx] with compile-time indexing only (keeps the key array in registers)
template <int NK>
__device__ __forceinline__ uint64_t pick(const uint64_t (&x)[NK], uint32_t idx) {
    uint64_t v = x[0];
#pragma unroll
    for (int k = 1; k < NK; ++k)
        if (idx == (uint32_t)k) v = x[k];
    return v;
}

// all lanes: lane i < n applies buffered miss i (key x, count c) to every non-privatised
// 1-D sketch hashed on key column k
__device__ __forceinline__ void flush_misses(const SParams &P, const uint64_t *seeds, const uint64_t *mx, const int *mc,
                                             uint32_t n, uint32_t k) {
    const int lane = threadIdx.x & 31;
    if ((uint32_t)lane < n) {
        const uint64_t xv = mx[lane];
        const int cv = mc[lane];
        for (uint32_t tm = P.key[k].glob1d; tm; tm &= tm - 1) {
            const STarget &tg = P.tgt[__ffs(tm) - 1];
            update_1d(tg, seeds + tg.seed_off, nullptr, xv, cv);
        }
    }
    __syncwarp();
}

// one warp-wide batch: lanes with `valid` hold one surviving tuple each, canonical keys x[k]
template <int NK>
__device__ __forceinline__ void process_batch(const SParams &P, unsigned char *smem, bool valid, const uint64_t (&x)[NK]) {
    const uint32_t act = __ballot_sync(0xffffffffu, valid);
    if (!act) return;
    int32_t *sc = reinterpret_cast<int32_t *>(smem + P.off_sc);
    const uint64_t *seeds = reinterpret_cast<const uint64_t *>(smem + P.off_seed);
    const int lane = threadIdx.x & 31;
    bool la = false, lb = false;   // trio keys: this lane leads its key group (size ca / cb)
    int ca = 0, cb = 0;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        if (!P.key[k].has1d) continue;
        // aggregate equal keys of the warp (match_any); the leader updates with the count
        bool leader = false, miss = false;
        int cnt = 0;
        if (valid) {
            const uint32_t grp = __match_any_sync(act, x[k]);
            leader = lane == __ffs(grp) - 1;
            cnt = __popc(grp);
        }
        if (P.trio_on) {
            if ((uint32_t)k == P.trio_ka) { la = leader; ca = cnt; }
            if ((uint32_t)k == P.trio_kb) { lb = leader; cb = cnt; }
        }
        // histogram keys: the CTA stops probing the heavy-hitter table once it no longer pays
        // (fewer than 1 hit in 4 probes after 8192 probes: a flat key distribution); what the
        // table holds is still flushed at the end, so the counts stay exact either way
        uint32_t *hstat = reinterpret_cast<uint32_t *>(smem + P.off_hstat) + k * 4;
        // the flag is written concurrently by other warps: lane 0's read is broadcast so the
        // full-mask ballots below are reached by every lane or by none (warp-uniform branch)
        uint32_t hh_off_flag = 0;
        if (P.key[k].hist && P.key[k].hh_off >= 0)
            hh_off_flag = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t *>(hstat + 2), 0);
        const bool use_hh = P.key[k].hh_off >= 0 && (!P.key[k].hist || hh_off_flag == 0);
        bool hh_hit = false;
        if (leader) {
            if (P.key[k].hist) {
                // histogram mode: count the key (heavy-hitter table first, then the L2 histogram);
                // all 1-D sketches of this key are built from the counts after the scan
                bool done = use_hh && hh_add(smem + P.key[k].hh_off, P.hh_log2, x[k], cnt);
                hh_hit = done;
                if (!done && x[k] < P.key[k].domain) { red_add_u32(P.key[k].hist + x[k], (uint32_t)cnt); done = true; }
                if (!done) {   // outside the hinted domain: direct updates
                    miss = P.key[k].hasglob;
                    for (uint32_t tm = P.key[k].priv1d; tm; tm &= tm - 1) {
                        const STarget &tg = P.tgt[__ffs(tm) - 1];
                        update_1d(tg, seeds + tg.seed_off, sc, x[k], cnt);
                    }
                }
            } else {
                if (P.key[k].hh_off >= 0) miss = !hh_add(smem + P.key[k].hh_off, P.hh_log2, x[k], cnt);
                else miss = P.key[k].hasglob;
                for (uint32_t tm = P.key[k].priv1d; tm; tm &= tm - 1) {   // privatised: always direct
                    const STarget &tg = P.tgt[__ffs(tm) - 1];
                    update_1d(tg, seeds + tg.seed_off, sc, x[k], cnt);
                }
            }
        }
        if (P.key[k].hist && use_hh) {
            const uint32_t np = __popc(__ballot_sync(0xffffffffu, leader));
            const uint32_t nh = __popc(__ballot_sync(0xffffffffu, hh_hit));
            if (lane == 0 && np) {
                const uint32_t p0 = atomicAdd(hstat, np), h0 = atomicAdd(hstat + 1, nh);
                if (p0 + np >= 8192 && (h0 + nh) * 4 < p0 + np) hstat[2] = 1;
            }
        }
        if (P.key[k].hasglob) {
            // keys without a heavy-hitter slot go to this warp's miss buffer; 32 buffered
            // misses are flushed together so every lane hashes (SIMT-efficient L2 updates)
            const uint32_t mb = __ballot_sync(0xffffffffu, miss);
            if (mb) {
                const uint32_t mi = (threadIdx.x >> 5) * P.n_keys + k;
                uint64_t *mx = reinterpret_cast<uint64_t *>(smem + P.off_miss) + mi * 32;
                int *mc = reinterpret_cast<int *>(smem + P.off_miss + kWarps * P.n_keys * 32 * 8) + mi * 32;
                uint32_t *nm = reinterpret_cast<uint32_t *>(smem + P.off_missn) + mi;
                uint32_t fill = *nm;
                const uint32_t nnew = __popc(mb);
                if (fill + nnew > 32) {
                    __syncwarp();
                    flush_misses(P, seeds, mx, mc, fill, (uint32_t)k);
                    fill = 0;
                }
                if (miss) {
                    const uint32_t pos = fill + __popc(mb & ((1u << lane) - 1u));
                    mx[pos] = x[k];
                    mc[pos] = cnt;
                }
                __syncwarp();
                if (lane == 0) *nm = fill + nnew;
                __syncwarp();
            }
        }
    }
    // matrix targets: equal key pairs of the warp aggregated (two match_any), the leader
    // updates one cell per row with count * xi * xi
    if (valid && P.has2d) {
        for (uint32_t t = 0; t < P.n_targets; ++t) {
            const STarget &tg = P.tgt[t];
            if (tg.ndim != 2 || (P.trio_on && t == P.trio_m)) continue;
            const uint64_t xa = pick<NK>(x, tg.k0), xb = pick<NK>(x, tg.k1);
            const uint32_t grp = __match_any_sync(act, xa) & __match_any_sync(act, xb);
            if (lane == __ffs(grp) - 1) update_2d(tg, seeds + tg.seed_off, sc, xa, xb, __popc(grp));
        }
    }
    if (valid && P.trio_on) {
        const uint64_t xa = pick<NK>(x, P.trio_ka), xb = pick<NK>(x, P.trio_kb);
        const uint32_t grp = __match_any_sync(act, xa) & __match_any_sync(act, xb);
        const bool lm = lane == __ffs(grp) - 1;
        const int cm = __popc(grp);
        if (la || lb || lm) {
            const STarget &A = P.tgt[P.trio_a], &B = P.tgt[P.trio_b], &M = P.tgt[P.trio_m];
            const uint64_t *sa = seeds + A.seed_off, *sb = seeds + B.seed_off;
            const bool narrow = (xa | xb) < (1ULL << 32);
            for (uint32_t r = 0; r < M.d; ++r) {
                const uint64_t *a = sa + r * 6, *b = sb + r * 6;
                uint32_t ga, gb;
                int xia, xib;
                if (narrow) {
                    ga = (uint32_t)hash_g61_t<true>(a[4], a[5], xa);
                    gb = (uint32_t)hash_g61_t<true>(b[4], b[5], xb);
                    xia = xi_sign61_t<true>(a, xa);
                    xib = xi_sign61_t<true>(b, xb);
                } else {
                    ga = (uint32_t)hash_g61_t<false>(a[4], a[5], xa);
                    gb = (uint32_t)hash_g61_t<false>(b[4], b[5], xb);
                    xia = xi_sign61_t<false>(a, xa);
                    xib = xi_sign61_t<false>(b, xb);
                }
                if (la) atomicAdd(&sc[A.smem_off + r * A.cells + (ga & A.wmask0)], xia * ca);
                if (lb) atomicAdd(&sc[B.smem_off + r * B.cells + (gb & B.wmask0)], xib * cb);
                if (lm) {
                    const uint32_t cell = ((ga & M.wmask0) << M.lw1) | (gb & M.wmask1);
                    const int v = xia * xib * cm;
                    if (M.smem_off >= 0) atomicAdd(&sc[M.smem_off + r * M.cells + cell], v);
                    else red_add_s64(M.counters + uint64_t(r) * M.cells + cell, (int64_t)v);
                }
            }
        }
    }
}

// register copy of one predicate (A2)
struct PR {
    uint32_t kind, bytes, n;
    int32_t soff;
    int64_t lo;
    uint64_t span;
    const void *p;
    const int64_t *set;
};

// conjunction of the predicates over this lane's 4 rows r0..r0+3 -> m[j] (A2).  FULL: the
// rows come from the staged tile (128-bit shared loads); otherwise from global memory,
// rows past the end are false.  R32: every predicate is an int32 range (no kind branches):
// one unsigned subtract-compare per row, ANDed into a predicate register.
template <int NP, bool R32, bool FULL>
__device__ __forceinline__ void eval_preds(const PR (&pr)[NP], const unsigned char *stage, uint64_t row0, int r0,
                                           int valid, bool (&m)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = FULL || j < valid;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        if (R32 || pr[q].kind == PR_R32) {
            int4 v;
            if (FULL) v = *reinterpret_cast<const int4 *>(stage + pr[q].soff + r0 * 4);
            else {
                const int *g = reinterpret_cast<const int *>(pr[q].p) + row0 + r0;
                v.x = valid > 0 ? __ldg(g) : 0; v.y = valid > 1 ? __ldg(g + 1) : 0;
                v.z = valid > 2 ? __ldg(g + 2) : 0; v.w = valid > 3 ? __ldg(g + 3) : 0;
            }
            const uint32_t lo = (uint32_t)pr[q].lo, sp = (uint32_t)pr[q].span;
            m[0] = m[0] & ((uint32_t)v.x - lo <= sp);
            m[1] = m[1] & ((uint32_t)v.y - lo <= sp);
            m[2] = m[2] & ((uint32_t)v.z - lo <= sp);
            m[3] = m[3] & ((uint32_t)v.w - lo <= sp);
        } else if (pr[q].kind == PR_R64) {
            int64_t v[4];
            if (FULL) {
                const longlong2 a = *reinterpret_cast<const longlong2 *>(stage + pr[q].soff + r0 * 8);
                const longlong2 b = *reinterpret_cast<const longlong2 *>(stage + pr[q].soff + r0 * 8 + 16);
                v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
            } else {
                const long long *g = reinterpret_cast<const long long *>(pr[q].p) + row0 + r0;
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = j < valid ? __ldg(g + j) : 0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) m[j] = m[j] & ((uint64_t)v[j] - (uint64_t)pr[q].lo <= pr[q].span);
        } else if (pr[q].kind == PR_SET) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (!m[j]) continue;
                int64_t v;
                if (FULL) v = pr[q].bytes == 8 ? *reinterpret_cast<const int64_t *>(stage + pr[q].soff + (r0 + j) * 8)
                                               : (int64_t) * reinterpret_cast<const int *>(stage + pr[q].soff + (r0 + j) * 4);
                else v = pr[q].bytes == 8 ? __ldg(reinterpret_cast<const long long *>(pr[q].p) + row0 + r0 + j)
                                          : (int64_t)__ldg(reinterpret_cast<const int *>(pr[q].p) + row0 + r0 + j);
                m[j] = in_set(pr[q].set, pr[q].n, v);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) m[j] = false;
        }
    }
}

// A3: one sector-granular gather of a survivor's key into the ring; the copy size (4 or 8
// bytes) is chosen by a predicate so one address computation serves both key widths
__device__ __forceinline__ void cp_async_key(uint32_t dst, const void *src, uint32_t is8) {
    asm volatile(
        "{\n\t.reg .pred p8;\n\tsetp.ne.u32 p8, %2, 0;\n\t"
        "@p8 cp.async.ca.shared.global.L2::64B [%0], [%1], 8;\n\t"
        "@!p8 cp.async.ca.shared.global.L2::64B [%0], [%1], 4;\n}" ::"r"(dst), "l"(src), "r"(is8)
        : "memory");
}
template <int W>
__device__ __forceinline__ void cp_async_fixed_if(bool on, uint32_t dst, const void *src) {
    if (W == 8)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                     "@p cp.async.ca.shared.global.L2::64B [%0], [%1], 8;\n}" ::"r"(dst), "l"(src), "r"((int)on)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                     "@p cp.async.ca.shared.global.L2::64B [%0], [%1], 4;\n}" ::"r"(dst), "l"(src), "r"((int)on)
                     : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}

template <int NK>
__device__ __forceinline__ void drain_batch(const SParams &P, unsigned char *smem, const unsigned char *q,
                                            const uint32_t (&kbytes)[NK], uint32_t head, uint32_t n) {
#ifdef SCAN_NOHASH   // timing experiments only (tools/build_variant.sh): results are wrong
    return;
#endif
    const int lane = threadIdx.x & 31;
    const bool valid = (uint32_t)lane < n;
    uint64_t xk[NK];
    const unsigned char *e = q + ((head + lane) & (P.cap - 1)) * (NK * 8);
#pragma unroll
    for (int k = 0; k < NK; ++k)
        xk[k] = valid ? canon61(kbytes[k] == 8 ? *reinterpret_cast<const int64_t *>(e + k * 8)
                                               : (int64_t) * reinterpret_cast<const int32_t *>(e + k * 8))
                      : 0;
    process_batch<NK>(P, smem, valid, xk);
}

// KW = 0: generic (any predicate kinds, key widths read at run time); KW = 4 / 8: every
// predicate is an int32 range and every key column is KW bytes wide (no kind or width
// branches; survivors' keys are gathered straight from the ballots)
template <int NK, int NP, int KW>
__global__ void __launch_bounds__(kThreads, 1) k_scan(const __grid_constant__ SParams P) {
    constexpr bool R32 = KW != 0;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full_all = reinterpret_cast<uint64_t *>(smem);   // [kGroups][kMaxStages]
    uint64_t *empty_all = full_all + kGroups * kMaxStages;     // [kGroups][kMaxStages]
    const uint32_t kStages = P.stages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ring group of this warp (producers are warps kWarps .. kWarps + kGroups - 1)
    const int grp = warp < kWarps ? warp / kGW : warp - kWarps;
    uint64_t *full = full_all + grp * kMaxStages, *empty = empty_all + grp * kMaxStages;
    const uint32_t G = gridDim.x * kGroups, gid = blockIdx.x * kGroups + grp;   // this group's tiles: gid + k*G

    // ---- setup: barriers, smem counters, heavy-hitter tables, seeds
    if (tid == 0) {
        for (uint32_t s = 0; s < kGroups * kMaxStages; ++s) { mbar_init(&full_all[s], 1); mbar_init(&empty_all[s], kGW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {
        int32_t *sc = reinterpret_cast<int32_t *>(smem + P.off_sc);
        for (uint32_t i = tid; i < P.smem_counters; i += kThreads) sc[i] = 0;
        for (uint32_t k = 0; k < P.n_keys; ++k) {
            if (P.key[k].hh_off < 0) continue;
            uint64_t *keys = reinterpret_cast<uint64_t *>(smem + P.key[k].hh_off);
            int *cnts = reinterpret_cast<int *>(smem + P.key[k].hh_off + (8u << P.hh_log2));
            for (uint32_t i = tid; i < (1u << P.hh_log2); i += kThreads) { keys[i] = kEmpty; cnts[i] = 0; }
        }
        uint64_t *sseed = reinterpret_cast<uint64_t *>(smem + P.off_seed);
        for (uint32_t t = 0; t < P.n_targets; ++t) {
            const uint32_t words = P.tgt[t].ndim * P.tgt[t].d * 6;
            for (uint32_t i = tid; i < words; i += kThreads) sseed[P.tgt[t].seed_off + i] = P.seeds[t][i];
        }
        uint32_t *nm = reinterpret_cast<uint32_t *>(smem + P.off_missn);
        for (uint32_t i = tid; i < kWarps * P.n_keys; i += kThreads) nm[i] = 0;
        uint32_t *hs = reinterpret_cast<uint32_t *>(smem + P.off_hstat);
        for (uint32_t i = tid; i < kMaxKeys * 4; i += kThreads) hs[i] = 0;
    }
    __syncthreads();

    if (warp >= kWarps) {
        // ================= producer warp of ring group grp: TMA bulk copies of staged columns
        if (lane == 0) {
            uint32_t s = 0, ph = 0;
            bool wrapped = false;
            for (uint64_t t = gid; t < P.n_tiles; t += G) {
                if (wrapped) mbar_wait(&empty[s], ph ^ 1);
                const uint64_t row0 = t * P.tile_rows;
                const bool fulltile = row0 + P.tile_rows <= P.n_rows;
                if (fulltile && P.stage_bytes) {
                    mbar_arrive_tx(&full[s], P.stage_bytes);
                    unsigned char *stage = smem + P.off_ring + (grp * kStages + s) * P.stage_bytes;
                    for (uint32_t c = 0; c < P.n_cols; ++c) {
                        if (P.col[c].soff < 0) continue;
                        const uint32_t b = P.col[c].bytes;
                        bulk_g2s(stage + P.col[c].soff, reinterpret_cast<const unsigned char *>(P.col[c].p) + row0 * b,
                                 P.tile_rows * b, &full[s]);
                    }
                } else {
                    mbar_arrive(&full[s]);
                }
                if (++s == kStages) { s = 0; ph ^= 1; wrapped = true; }
            }
        }
        return;
    }

    // ================= consumer warps: independent pipelines, no CTA-wide barrier in the loop
    PR pr[(NP > 0) ? NP : 1];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const SPred &sp = P.pred[q];
        const SCol &c = P.col[sp.col];
        pr[q] = PR{sp.kind, c.bytes, sp.n, c.soff, sp.lo, sp.span, c.p, sp.set};
    }
    const void *kptr[NK];
    uint32_t kbytes[NK];
    int32_t ksoff[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const SCol &c = P.col[P.key[k].col];
        kptr[k] = c.p;
        kbytes[k] = c.bytes;
        ksoff[k] = c.soff;
    }
    const uint32_t cap = P.cap;
    uint32_t surv = 0;                       // warp-uniform exact survivor count
    const int r0 = (warp % kGW) * 128 + lane * 4;   // this lane's 4 rows inside its group's tile
    unsigned char *q = smem + P.off_kbuf + warp * P.kb_bytes;   // this warp's survivor-key ring
    const uint32_t q_a = smem_u32(q);
    const uint32_t rl_a = smem_u32(smem + P.off_rows) + warp * 256;   // this warp's survivor row list
    uint32_t head = 0, tail = 0;             // ring positions (monotone)
    uint32_t tl[kLag];                       // ring tail after each of the previous kLag tiles
#pragma unroll
    for (int i = 0; i < kLag; ++i) tl[i] = 0;
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t n_tiles = (uint32_t)P.n_tiles;
    constexpr int NPX = (NP > 0) ? NP : 1;
    uint32_t s = 0, ph = 0;
    for (uint32_t t = gid; t < n_tiles; t += G) {
        const uint64_t row0 = uint64_t(t) * kTile;
        mbar_wait_a(full_a + s * 8, ph);
        const unsigned char *stage = smem + P.off_ring + (grp * kStages + s) * P.stage_bytes;
        const bool full_tile = t < P.n_full_tiles;   // staged by the producer
        if (NP > 0) {
            bool m[4];
            if (full_tile) eval_preds<NPX, R32, true>(pr, stage, row0, r0, 4, m);
            else {
                const int64_t rem = (int64_t)P.n_rows - (int64_t)(row0 + r0);
                eval_preds<NPX, R32, false>(pr, stage, row0, r0, rem <= 0 ? 0 : (rem >= 4 ? 4 : (int)rem), m);
            }
            // one ballot per row slot; the ballots also order every lane's shared reads of
            // stage s before lane 0 releases it
            const uint32_t B0 = __ballot_sync(0xffffffffu, m[0]), B1 = __ballot_sync(0xffffffffu, m[1]);
            const uint32_t B2 = __ballot_sync(0xffffffffu, m[2]), B3 = __ballot_sync(0xffffffffu, m[3]);
            if (lane == 0) mbar_arrive_a(empty_a + s * 8);
            const uint32_t c0 = __popc(B0), c1 = __popc(B1), c2 = __popc(B2), c3 = __popc(B3);
            const uint32_t wtot = c0 + c1 + c2 + c3;
            surv += wtot;
            if (wtot) {
                if (KW != 0 && tail - head + wtot <= cap) {
                    // survivors in slot-major order (slot j of every lane, then slot j+1): ring
                    // position = popc of one ballot, gathered straight from the owning lane
                    const uint32_t pb[4] = {tail, tail + c0, tail + c0 + c1, tail + c0 + c1 + c2};
                    const uint32_t bj[4] = {B0, B1, B2, B3};
                    const unsigned char *kb[NK];
#pragma unroll
                    for (int k = 0; k < NK; ++k)
                        kb[k] = reinterpret_cast<const unsigned char *>(kptr[k]) + (row0 + r0) * (uint64_t)(KW ? KW : 8);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {   // predicated copies: no branches
                        const uint32_t dst = q_a + ((pb[j] + __popc(bj[j] & lt)) & (cap - 1)) * (NK * 8);
#pragma unroll
                        for (int k = 0; k < NK; ++k)
                            cp_async_fixed_if<KW ? KW : 8>(m[j], dst + k * 8, kb[k] + j * (KW ? KW : 8));
                    }
                    tail += wtot;
                } else {
                    // generic / ring-full path: each survivor's tile offset goes to the warp's
                    // row list (same slot-major order), then the gathers run converged over the
                    // list, in rounds that fit the ring (a tile may hold more survivors than it)
                    if (m[0]) sts_u16(rl_a + 2 * __popc(B0 & lt), r0);
                    if (m[1]) sts_u16(rl_a + 2 * (c0 + __popc(B1 & lt)), r0 + 1);
                    if (m[2]) sts_u16(rl_a + 2 * (c0 + c1 + __popc(B2 & lt)), r0 + 2);
                    if (m[3]) sts_u16(rl_a + 2 * (c0 + c1 + c2 + __popc(B3 & lt)), r0 + 3);
                    __syncwarp();
                    for (uint32_t e0 = 0; e0 < wtot;) {
                        if (tail - head == cap || (e0 == 0 && tail - head + wtot > cap)) {
                            // ring would overflow: finish outstanding gathers and drain it completely
                            // (mid-tile, the gathers just issued are not committed yet)
                            if (e0 == 0) cp_wait_all();
                            else cp_commit_wait_all();
                            __syncwarp();
                            while (tail != head) {
                                const uint32_t n = min(32u, tail - head);
                                drain_batch<NK>(P, smem, q, kbytes, head, n);
                                head += n;
                            }
#pragma unroll
                            for (int i = 0; i < kLag; ++i) tl[i] = tail;
                        }
                        const uint32_t n = min(wtot - e0, cap - (tail - head));   // a tile may exceed cap
                        for (uint32_t e = lane; e < n; e += 32) {
                            const uint64_t row = row0 + lds_u16(rl_a + 2 * (e0 + e));
                            const uint32_t dst = q_a + ((tail + e) & (cap - 1)) * (NK * 8);
#ifndef SCAN_NOGATHER   // timing experiments only (tools/build_variant.sh): results are wrong
#pragma unroll
                            for (int k = 0; k < NK; ++k)
                                cp_async_key(dst + k * 8, reinterpret_cast<const unsigned char *>(kptr[k]) + row * kbytes[k],
                                             kbytes[k] == 8);
#endif
                        }
                        tail += n;
                        e0 += n;
                    }
                    __syncwarp();
                }
            }
            // one cp.async group per tile (possibly empty): wait_group kLag then guarantees the
            // entries appended kLag tiles ago (t3) have landed; the latency hides behind 3 tiles
            cp_commit();
            const uint32_t ready_end = tl[kLag - 1];
#pragma unroll
            for (int i = kLag - 1; i > 0; --i) tl[i] = tl[i - 1];
            tl[0] = tail;
            if (ready_end - head >= 32) {
                cp_wait_lag();
                __syncwarp();
                while (ready_end - head >= 32) { drain_batch<NK>(P, smem, q, kbytes, head, 32); head += 32; }
            }
        } else {
            // keys are staged (no predicate): aggregate and update straight from the stage
            const int64_t rem = (int64_t)P.n_rows - (int64_t)(row0 + r0);
            const int valid = rem <= 0 ? 0 : (rem >= 4 ? 4 : (int)rem);
            const uint32_t bits = (1u << valid) - 1u;
            surv += __reduce_add_sync(0xffffffffu, (uint32_t)valid);
            uint64_t xs[4][NK];
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                if (kbytes[k] == 4) {
                    int4 v;
                    if (full_tile) v = *reinterpret_cast<const int4 *>(stage + ksoff[k] + r0 * 4);
                    else {
                        const int *g = reinterpret_cast<const int *>(kptr[k]) + row0 + r0;
                        v.x = valid > 0 ? __ldg(g) : 0; v.y = valid > 1 ? __ldg(g + 1) : 0;
                        v.z = valid > 2 ? __ldg(g + 2) : 0; v.w = valid > 3 ? __ldg(g + 3) : 0;
                    }
                    xs[0][k] = canon61(v.x); xs[1][k] = canon61(v.y); xs[2][k] = canon61(v.z); xs[3][k] = canon61(v.w);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        int64_t v = 0;
                        if (full_tile) v = *reinterpret_cast<const int64_t *>(stage + ksoff[k] + (r0 + j) * 8);
                        else if (j < valid) v = __ldg(reinterpret_cast<const long long *>(kptr[k]) + row0 + r0 + j);
                        xs[j][k] = canon61(v);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) process_batch<NK>(P, smem, (bits >> j) & 1u, xs[j]);
            __syncwarp();
            if (lane == 0) mbar_arrive_a(empty_a + s * 8);
        }
        if (++s == kStages) { s = 0; ph ^= 1; }
    }
    if (NP > 0) {
        cp_wait_all();
        __syncwarp();
        while (tail - head > 0) {
            const uint32_t n = min(32u, tail - head);
            drain_batch<NK>(P, smem, q, kbytes, head, n);
            head += n;
        }
    }

    // ---- this warp's buffered heavy-hitter misses
    {
        const uint64_t *seeds = reinterpret_cast<const uint64_t *>(smem + P.off_seed);
        __syncwarp();
        for (uint32_t k = 0; k < P.n_keys; ++k) {
            if (!P.key[k].hasglob) continue;
            const uint32_t mi = warp * P.n_keys + k;
            const uint32_t n = reinterpret_cast<volatile uint32_t *>(smem + P.off_missn)[mi];
            if (n) flush_misses(P, seeds, reinterpret_cast<const uint64_t *>(smem + P.off_miss) + mi * 32,
                                reinterpret_cast<const int *>(smem + P.off_miss + kWarps * P.n_keys * 32 * 8) + mi * 32, n, k);
        }
    }
    // ---- exact survivor count
    if (lane == 0 && surv && P.survivors) atomicAdd(P.survivors, (unsigned long long)surv);
    consumer_sync();
    // ---- flush heavy-hitter tables (one hash evaluation per distinct key per CTA)
    int32_t *sc = reinterpret_cast<int32_t *>(smem + P.off_sc);
    const uint64_t *seeds = reinterpret_cast<const uint64_t *>(smem + P.off_seed);
    for (uint32_t k = 0; k < P.n_keys; ++k) {
        if (P.key[k].hh_off < 0) continue;
        const uint64_t *keys = reinterpret_cast<const uint64_t *>(smem + P.key[k].hh_off);
        const int *cnts = reinterpret_cast<const int *>(smem + P.key[k].hh_off + (8u << P.hh_log2));
        for (uint32_t s = tid; s < (1u << P.hh_log2); s += kConsumers) {
            const uint64_t x = keys[s];
            const int c = cnts[s];
            if (x == kEmpty || c == 0) continue;
            if (P.key[k].hist) {
                if (x < P.key[k].domain) { red_add_u32(P.key[k].hist + x, (uint32_t)c); continue; }
                for (uint32_t tt = 0; tt < P.n_targets; ++tt) {   // outside the domain: all targets directly
                    const STarget &tg = P.tgt[tt];
                    if (tg.ndim != 1 || tg.k0 != k) continue;
                    update_1d(tg, seeds + tg.seed_off, sc, x, c);
                }
                continue;
            }
            for (uint32_t tt = 0; tt < P.n_targets; ++tt) {
                const STarget &tg = P.tgt[tt];
                if (tg.ndim != 1 || tg.k0 != k || tg.smem_off >= 0) continue;
                update_1d(tg, seeds + tg.seed_off, sc, x, c);
            }
        }
    }
    consumer_sync();
    // ---- flush privatised int32 counters into the int64 sketches
    for (uint32_t tt = 0; tt < P.n_targets; ++tt) {
        const STarget &tg = P.tgt[tt];
        if (tg.smem_off < 0) continue;
        const uint32_t n = tg.d * tg.cells;
        for (uint32_t qq = tid; qq < n; qq += kConsumers) {
            const int32_t v = sc[tg.smem_off + qq];
            if (v) red_add_s64(tg.counters + qq, (int64_t)v);
        }
    }
}

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

typedef void (*ScanKernel)(const SParams);

template <int NK, int NP>
static ScanKernel pick_kw(int kw) {
    if (NP == 0) return k_scan<NK, NP, 0>;
    return kw == 4 ? k_scan<NK, NP, 4> : kw == 8 ? k_scan<NK, NP, 8> : k_scan<NK, NP, 0>;
}

template <int NK>
static ScanKernel pick_np(uint32_t np, int kw) {
    switch (np) {
        case 0: return pick_kw<NK, 0>(kw);
        case 1: return pick_kw<NK, 1>(kw);
        case 2: return pick_kw<NK, 2>(kw);
        case 3: return pick_kw<NK, 3>(kw);
        default: return pick_kw<NK, 4>(kw);
    }
}

static ScanKernel pick_kernel(uint32_t nk, uint32_t np, int kw) {
    switch (nk) {
        case 1: return pick_np<1>(np, kw);
        case 2: return pick_np<2>(np, kw);
        case 3: return pick_np<3>(np, kw);
        default: return pick_np<4>(np, kw);
    }
}

}  // namespace

namespace skb {

// Returns SK_OK and sets *launched if the optimised scan handled the call; leaves
// *launched false (and returns SK_OK) when the call is outside its envelope.
sk_status scan_launch(const ScanCall &c, cudaStream_t stream, bool *launched) {
    *launched = false;
    if (c.n_cols > kMaxSCols || c.n_preds > 4 || c.n_targets > kMaxSTargets || c.n_rows == 0) return SK_OK;
    SParams P;
    memset(&P, 0, sizeof(P));
    P.n_cols = c.n_cols;
    P.n_rows = c.n_rows;
    for (uint32_t i = 0; i < c.n_cols; ++i) {
        P.col[i].p = c.col_ptr[i];
        P.col[i].bytes = c.col_bytes[i];
        P.col[i].soff = -1;
        if (((uintptr_t)c.col_ptr[i]) & 15) return SK_OK;   // bulk copies need 16-byte alignment
    }
    // distinct key columns
    std::vector<uint32_t> keys;
    for (uint32_t t = 0; t < c.n_targets; ++t)
        for (uint32_t q = 0; q < c.tgt_ndim[t]; ++q)
            if (std::find(keys.begin(), keys.end(), c.tgt_key[t][q]) == keys.end()) keys.push_back(c.tgt_key[t][q]);
    if (keys.size() > (size_t)kMaxKeys) return SK_OK;
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
    P.gather = c.n_preds > 0 ? 1u : 0u;
    P.tile_rows = kTile;
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
            return SK_OK;
        }
    }
    // ---- shared-memory plan (227 KB): barriers | TMA ring (stages x stage) | per-warp key
    //      rings | privatised counters | heavy-hitter tables | seeds.  Tunables via env
    //      (COMPASS_STAGES, COMPASS_HH_LOG2) for experiments only.
    const uint32_t kBudget = 227 * 1024;
    const char *env_st = getenv("COMPASS_STAGES"), *env_hh = getenv("COMPASS_HH_LOG2");
    const uint32_t want_stages = env_st ? (uint32_t)atoi(env_st) : 6;
    const uint32_t max_hh = env_hh ? (uint32_t)atoi(env_hh) : 11;
    uint32_t seed_words = 0;
    for (uint32_t t = 0; t < c.n_targets; ++t) seed_words += c.tgt_ndim[t] * c.tgt_d[t] * 6;
    P.seed_words = seed_words;
    const uint32_t seed_bytes = (seed_words * 8 + 15) & ~15u;
    for (uint32_t k = 0; k < P.n_keys; ++k) P.key[k].col = keys[k];
    P.cap = 0;
    P.kb_bytes = 0;
    const uint32_t ring_warps = kWarps;                 // warps owning a survivor-key ring
    if (P.gather) {
        P.cap = P.n_keys == 1 ? 256 : SCAN_CAP2;              // >= one tile-slice of survivors (128); overflow drains
        P.kb_bytes = P.cap * P.n_keys * 8;
    }
    const uint32_t min_stages = 3;
    const uint32_t miss_bytes = kWarps * P.n_keys * 32 * 12 + ((kWarps * P.n_keys * 4 + 15) & ~15u) + kMaxKeys * 16 + 16;
    const uint32_t kBarBytes = 2 * kGroups * kMaxStages * 8;
    const uint32_t ring_stage = kGroups * P.stage_bytes;   // one stage of every group's ring
    const uint32_t fixed = kBarBytes + min_stages * ring_stage + ring_warps * P.kb_bytes + seed_bytes + miss_bytes +
                           kWarps * 128 * 2 + 256;
    if (fixed > kBudget) return SK_OK;
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
        tg.wmask1 = tg.ndim == 2 ? c.tgt_w[t][1] - 1 : 0;
        tg.lw1 = tg.ndim == 2 ? (uint32_t)__builtin_ctz(c.tgt_w[t][1]) : 0;
        tg.k0 = (uint32_t)(std::find(keys.begin(), keys.end(), c.tgt_key[t][0]) - keys.begin());
        tg.k1 = tg.ndim == 2 ? (uint32_t)(std::find(keys.begin(), keys.end(), c.tgt_key[t][1]) - keys.begin()) : 0;
        tg.cells = tg.ndim == 2 ? c.tgt_w[t][0] * c.tgt_w[t][1] : c.tgt_w[t][0];
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
        if (tg.ndim == 2) P.has2d = 1;
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
    // hash lookup tables for matrix dimensions whose key column has a domain hint (the table
    // stays L2-resident: dom * d * 4 bytes <= 64 MB per dimension); built once per sketch
    if (!(getenv("COMPASS_LUT") && strcmp(getenv("COMPASS_LUT"), "0") == 0)) {
        int dev_l = 0, sms_l = 148;
        cudaGetDevice(&dev_l);
        cudaDeviceGetAttribute(&sms_l, cudaDevAttrMultiProcessorCount, dev_l);
        for (uint32_t t = 0; t < c.n_targets; ++t) {
            STarget &tg = P.tgt[t];
            tg.lut0 = tg.lut1 = nullptr;
            if (tg.ndim != 2 || !c.tgt_sketch[t]) continue;
            sk_sketch *sk = c.tgt_sketch[t];
            const uint64_t dom[2] = {c.col_domain[c.tgt_key[t][0]], c.col_domain[c.tgt_key[t][1]]};
            bool ok = true;
            const uint64_t dp = (sk->d + 3) & ~3u;
            for (int q = 0; q < 2; ++q) ok &= sk->d <= 8 && dom[q] > 0 && dom[q] <= (1ULL << 31) && dom[q] * dp * 4 <= (64ULL << 20);
            if (!ok) continue;
            std::lock_guard<std::mutex> lk(sk->lut_mu);
            bool built = false;
            for (int q = 0; q < 2; ++q) {
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
            tg.lut_dom0 = dom[0];
            tg.lut_dom1 = dom[1];
        }
    }
    // trio detection: matrix M whose dimension-q hash rows equal those of a privatised 1-D
    // sketch on the same key (exact comparison of the coefficient rows; same d)
    P.trio_on = 0;
    for (uint32_t m = 0; m < c.n_targets && !P.trio_on; ++m) {
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
    while (stages < kMaxStages && !env_st && avail >= ring_stage && nhh == 0) { ++stages; avail -= ring_stage; }
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
    P.off_hstat = (off + 15) & ~15u;
    off = P.off_hstat + kMaxKeys * 4 * 4;
    P.off_seed = (off + 15) & ~15u;
    off = P.off_seed + seed_bytes;
    if (off > kBudget) return SK_OK;
    P.survivors = c.survivors;

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t grid = std::min<uint64_t>((uint64_t)sms, (P.n_tiles + kGroups - 1) / kGroups);
    // int32 privatised counts stay exact: rows per CTA < 2^31
    if ((P.n_tiles + grid * kGroups - 1) / (grid * kGroups) * P.tile_rows * kGroups >= (1ULL << 31)) return SK_OK;
    if (P.n_keys == 0) return SK_OK;
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
    ScanKernel kern = pick_kernel(P.n_keys, P.n_preds, kw);
    const int threads = kThreads;
    if (getenv("COMPASS_SCAN_DEBUG"))
        fprintf(stderr, "k_scan plan: keys %u preds %u kw %d stages %u hh_log2 %u cap %u smem %u (ring %u, counters %u)\n",
                P.n_keys, P.n_preds, kw, P.stages, P.hh_log2, P.cap, off, P.stages * kGroups * P.stage_bytes,
                P.smem_counters * 4);
    SKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)off));
    kern<<<(unsigned)grid, threads, off, stream>>>(P);
    SKB_CUDA(cudaGetLastError());
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
