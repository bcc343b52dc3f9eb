// scan_kernel.cuh — device code of the optimised fused scan; see scan.cu
// for the design notes.  Included by scan.cu (host plan, epilogues) and by scan_k1..4.cu, which
// instantiate k_scan for 1..4 key columns in separate translation units (parallel builds).
#pragma once
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
#include "peer.cuh"
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
    uint32_t ndim, d, wmask0, wmask1, lw1, wmask2, lw2;
    uint32_t k0, k1, k2;  // indices into keys[]
    int32_t smem_off;     // int32 offset of privatised copy, -1 = global
    uint32_t cells;
    uint32_t seed_off;
    const uint32_t *lut0, *lut1, *lut2;   // matrices / tensors: per-dimension hash lookup tables (or null)
    uint64_t lut_dom0, lut_dom1, lut_dom2;
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
    uint32_t tile_rows;             // rows per ring stage (sub * kTile)
    uint32_t sub;                   // sub-tiles of kTile rows per stage (predicate path; 1 otherwise)
    uint32_t n_full_tiles;          // tiles with tile_rows rows (staged by TMA)
    unsigned long long *survivors;
    // fused cross-GPU merge (peer.cuh): after every CTA has flushed, the table's partial slice
    // is added into every rank's merged buffer (push.peers > 0 only in a cooperative launch)
    PeerPush push;
    unsigned int *push_bar;
    // lookup-table path (FAST instances): per key column, the lookup table of its hash family
    // over the hinted domain [0, klut_dom) (16 bytes per key: 8 uint16 fields, field r =
    // counter index r * w + bucket of the family's primary sketch << 1 | sign), the primary
    // sketch (the widest 1-D sketch of the family) and the other 1-D sketches on the column
    const uint4 *klut[kMaxKeys];
    uint64_t klut_dom[kMaxKeys];
    uint32_t n_mat, mat_t[2];        // matrix targets of the lookup-table path
    uint32_t kprim[kMaxKeys];
    uint32_t kothers[kMaxKeys];
    // skewed key pairs of one L2-backed matrix (target pair_t): a two-choice table of
    // (key pair -> count) at byte offset pairhh_off (-1 = none), 2^pair_log2 slots, used while
    // a warp aggregates (hot cells would otherwise serialise their L2 atomics)
    int32_t pairhh_off;
    uint32_t pair_log2, pair_t;
};

// Debug builds (-DCOMPASS_CHECKS, tools/build_variant.sh): device-side bounds checks on ring
// positions, staged-tile offsets and lookup-table counter indices; a violated check traps
// (a CUDA error at the next synchronisation), standing in for compute-sanitizer, which the
// gpurun pool does not allow.
#ifdef COMPASS_CHECKS
#define SCAN_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SCAN_CHECK(cond) do { } while (0)
#endif

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
// L2 prefetch size of the survivor-key gathers (experiments: tools/build_variant.sh
// -DSCAN_L2HINT='""')
#ifndef SCAN_L2HINT
#define SCAN_L2HINT ".L2::64B"
#endif
__device__ __forceinline__ void cp_wait_lag() { asm volatile("cp.async.wait_group %0;" ::"n"(kLag) : "memory"); }
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }
__device__ __forceinline__ void red_add_u32(uint32_t *p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_s64(int64_t *p, int64_t v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// shared-memory int32 add at a 32-bit shared address (no generic-to-shared conversion per update)
__device__ __forceinline__ void red_shared_s32(uint32_t a, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
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

// 3-D tensor target t: row r gets cnt * xi0(x) xi1(y) xi2(z) at cell
// [h0(x)][h1(y)][h2(z)], dimensions in the sketch's canonical edge order
template <bool N>
__device__ __forceinline__ void update_3d_t(const STarget &tg, const uint64_t *seed, int32_t *sc, uint64_t x, uint64_t y,
                                            uint64_t z, int cnt) {
    const uint64_t *s1 = seed + tg.d * 6, *s2 = s1 + tg.d * 6;
    for (uint32_t r = 0; r < tg.d; ++r) {
        const uint64_t *a = seed + r * 6, *b = s1 + r * 6, *c = s2 + r * 6;
        const uint32_t cell = ((((uint32_t)(hash_g61_t<N>(a[4], a[5], x) & tg.wmask0) << tg.lw1) |
                                (uint32_t)(hash_g61_t<N>(b[4], b[5], y) & tg.wmask1)) << tg.lw2) |
                              (uint32_t)(hash_g61_t<N>(c[4], c[5], z) & tg.wmask2);
        const int v = xi_sign61_t<N>(a, x) * xi_sign61_t<N>(b, y) * xi_sign61_t<N>(c, z) * cnt;
        if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + r * tg.cells + cell], v);
        else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, (int64_t)v);
    }
}
__device__ __forceinline__ void update_3d(const STarget &tg, const uint64_t *seed, int32_t *sc, uint64_t x, uint64_t y,
                                          uint64_t z, int cnt) {
    if (tg.lut0 && x < tg.lut_dom0 && y < tg.lut_dom1 && z < tg.lut_dom2) {
        // (bucket, sign) of every row of every dimension from the lookup tables, all loads
        // issued before the first update (same layout as update_2d)
        const uint32_t dp = (tg.d + 3) & ~3u;
        const uint4 *la = reinterpret_cast<const uint4 *>(tg.lut0 + x * dp), *lb = reinterpret_cast<const uint4 *>(tg.lut1 + y * dp),
                    *lc = reinterpret_cast<const uint4 *>(tg.lut2 + z * dp);
        uint4 va[2], vb[2], vc[2];
        va[0] = __ldg(la); vb[0] = __ldg(lb); vc[0] = __ldg(lc);
        if (dp > 4) { va[1] = __ldg(la + 1); vb[1] = __ldg(lb + 1); vc[1] = __ldg(lc + 1); }
        for (uint32_t r = 0; r < tg.d && r < 8; ++r) {
            const uint4 &qa = va[r >> 2], &qb = vb[r >> 2], &qc = vc[r >> 2];
            const uint32_t j = r & 3;
            const uint32_t ea = j == 0 ? qa.x : j == 1 ? qa.y : j == 2 ? qa.z : qa.w;
            const uint32_t eb = j == 0 ? qb.x : j == 1 ? qb.y : j == 2 ? qb.z : qb.w;
            const uint32_t ec = j == 0 ? qc.x : j == 1 ? qc.y : j == 2 ? qc.z : qc.w;
            const uint32_t cell = ((((ea >> 1) << tg.lw1) | (eb >> 1)) << tg.lw2) | (ec >> 1);
            const int v = ((ea ^ eb ^ ec) & 1u) ? -cnt : cnt;
            if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + r * tg.cells + cell], v);
            else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, (int64_t)v);
        }
        return;
    }
    if ((x | y | z) < (1ULL << 32)) update_3d_t<true>(tg, seed, sc, x, y, z, cnt);
    else update_3d_t<false>(tg, seed, sc, x, y, z, cnt);
}

// x[idx] with compile-time indexing only (keeps the key array in registers)
template <int NK, typename T>
__device__ __forceinline__ T pick(const T (&x)[NK], uint32_t idx) {
    T v = x[0];
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
template <int NK, bool T3>
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
            if (tg.ndim < 2 || (P.trio_on && t == P.trio_m)) continue;
            const uint64_t xa = pick<NK>(x, tg.k0), xb = pick<NK>(x, tg.k1);
            // 3-D tensor: equal key triples aggregated.  Only the T3 instances (launched when a
            // tensor target is present) carry this code: compiled into every hashing-drain
            // instance, it slowed the C4 scan (k_scan<2,3,8,0,1>, no tensor) from 2.9 to 5.0 ms
            if (T3 && tg.ndim == 3) {
                const uint64_t xc = pick<NK>(x, tg.k2);
                const uint32_t grp = __match_any_sync(act, xa) & __match_any_sync(act, xb) & __match_any_sync(act, xc);
                if (lane == __ffs(grp) - 1) update_3d(tg, seeds + tg.seed_off, sc, xa, xb, xc, __popc(grp));
                continue;
            }
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

// ------------------------------------------------------------------ lookup-table path
// FAST instances (every key column int32 with a hinted domain, one hash family per key
// column, d * (log2 w + 1) <= 64): a survivor's (bucket, sign) for every row of every
// sketch on a key column come from ONE 64-bit load of that column's packed lookup table
// (built once per sketch, L2-resident; the same values the hash polynomials give, H3/H4), so
// the drain does no hashing, no histogram and no heavy-hitter probing.  The load of batch
// k is issued before batch k-1 is applied (one batch pending per warp), hiding its latency.
// Matrix cells take the low bits of the 1-D family's buckets (h mod w_m = (h mod w) mod w_m,
// w_m | w).  Keys outside the hinted domain fall back to the hash polynomials.
template <int NK>
struct Pend {
    uint4 e[NK];
    int32_t x[NK];
    bool valid;
};

// field r (compile-time after unrolling) of a table entry
__device__ __forceinline__ uint32_t lut_fld(const uint4 &q, int r) {
    const uint32_t w = r < 2 ? q.x : (r < 4 ? q.y : (r < 6 ? q.z : q.w));
    return (r & 1) ? (w >> 16) : (w & 0xffffu);
}

template <int NK>
__device__ __forceinline__ void fast_load(const SParams &P, bool valid, const int32_t (&xr)[NK], Pend<NK> &n) {
    n.valid = valid;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        n.x[k] = xr[k];
        n.e[k] = (valid && (uint32_t)xr[k] < P.klut_dom[k]) ? __ldg(P.klut[k] + (uint32_t)xr[k]) : make_uint4(0, 0, 0, 0);
    }
}

// out-of-domain keys on the lookup-table path (rare): hashed by the polynomials (inlined: an
// out-of-line call made the kernel spill around it)
__device__ __forceinline__ void fast_slow_1d(const SParams &P, unsigned char *smem, uint32_t k, int32_t xr, int cnt) {
    int32_t *sc = reinterpret_cast<int32_t *>(smem + P.off_sc);
    const uint64_t *seeds = reinterpret_cast<const uint64_t *>(smem + P.off_seed);
    for (uint32_t tm = P.key[k].priv1d | P.key[k].glob1d; tm; tm &= tm - 1) {
        const STarget &tg = P.tgt[__ffs(tm) - 1];
        update_1d(tg, seeds + tg.seed_off, sc, canon61(xr), cnt);
    }
}
__device__ __forceinline__ void fast_slow_2d(const SParams &P, unsigned char *smem, uint32_t t, int32_t xa, int32_t xb, int cnt) {
    const STarget &tg = P.tgt[t];
    update_2d(tg, reinterpret_cast<const uint64_t *>(smem + P.off_seed) + tg.seed_off,
              reinterpret_cast<int32_t *>(smem + P.off_sc), canon61(xa), canon61(xb), cnt);
}

// apply one pending batch (all 32 lanes converged).  Key aggregation (match_any on the raw
// int32 keys, exact by linearity) is adaptive per warp: sampled once every 32
// batches and kept while at least 1/8 of the batch's lanes repeat a key (skewed columns).
template <int NK>
__device__ __forceinline__ void process_fast(const SParams &P, unsigned char *smem, const Pend<NK> &b, bool &agg,
                                             uint32_t &actr) {
    const uint32_t act = __ballot_sync(0xffffffffu, b.valid);
    if (!act) return;
    int32_t *sc = reinterpret_cast<int32_t *>(smem + P.off_sc);
    const uint64_t *seeds = reinterpret_cast<const uint64_t *>(smem + P.off_seed);
    const int lane = threadIdx.x & 31;
    uint32_t grp[NK];
    const bool do_match = agg || ((actr++ & 31u) == 0);
    if (do_match) {
#pragma unroll
        for (int k = 0; k < NK; ++k) grp[k] = b.valid ? __match_any_sync(act, (uint32_t)b.x[k]) : 0u;
        const uint32_t lead = __ballot_sync(0xffffffffu, b.valid && lane == __ffs(grp[0]) - 1);
        agg = (uint32_t)(__popc(act) - __popc(lead)) * 8u > (uint32_t)__popc(act);
    } else {
#pragma unroll
        for (int k = 0; k < NK; ++k) grp[k] = 1u << lane;
    }
    if (!b.valid) return;   // no warp collectives below
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        if (!P.key[k].has1d || lane != __ffs(grp[k]) - 1) continue;
        const int cnt = __popc(grp[k]);
        if ((uint32_t)b.x[k] >= P.klut_dom[k]) {   // outside the hinted domain: hash
            fast_slow_1d(P, smem, (uint32_t)k, b.x[k], cnt);
            continue;
        }
        const uint4 q = b.e[k];
        const STarget &tp = P.tgt[P.kprim[k]];   // field >> 1 is its counter index
        if (tp.smem_off >= 0) {
            const uint32_t base = smem_u32(sc + tp.smem_off);
            if (tp.d == 5) {   // the common depth: no per-row bound checks
#pragma unroll
                for (int r = 0; r < 5; ++r) {
                    const uint32_t f = lut_fld(q, r);
                    SCAN_CHECK((f >> 1) < tp.d * tp.cells && (f >> 1) / tp.cells == (uint32_t)r);
                    red_shared_s32(base + (f >> 1) * 4u, (f & 1u) ? -cnt : cnt);
                }
            } else {
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (r < (int)tp.d) {
                        const uint32_t f = lut_fld(q, r);
                        SCAN_CHECK((f >> 1) < tp.d * tp.cells && (f >> 1) / tp.cells == (uint32_t)r);
                        red_shared_s32(base + (f >> 1) * 4u, (f & 1u) ? -cnt : cnt);
                    }
            }
        } else {
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < (int)tp.d) {
                    const uint32_t f = lut_fld(q, r);
                    red_add_s64(tp.counters + (f >> 1), (f & 1u) ? -cnt : cnt);
                }
        }
        for (uint32_t tm = P.kothers[k]; tm; tm &= tm - 1) {   // narrower sketches of the family
            const STarget &tg = P.tgt[__ffs(tm) - 1];
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < (int)tg.d) {
                    const uint32_t f = lut_fld(q, r);
                    const uint32_t cell = (f >> 1) & tg.wmask0;
                    const int v = (f & 1u) ? -cnt : cnt;
                    if (tg.smem_off >= 0) atomicAdd(&sc[tg.smem_off + r * tg.cells + cell], v);
                    else red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, (int64_t)v);
                }
        }
    }
    for (uint32_t mi = 0; mi < P.n_mat; ++mi) {   // the matrix targets (at most two on this path)
        const uint32_t t = P.mat_t[mi];
        const STarget &tg = P.tgt[t];
        // NK <= 2 and a matrix spans both key columns (k0 = 0, k1 = 1 or the reverse)
        const bool swap = NK > 1 && tg.k0 != 0;
        const uint32_t g = NK > 1 ? (grp[0] & grp[NK - 1]) : grp[0];
        if (lane != __ffs(g) - 1) continue;
        const int cnt = __popc(g);
        const int32_t xa = swap ? b.x[NK - 1] : b.x[0], xb = swap ? b.x[0] : b.x[NK - 1];
        if ((uint32_t)xa >= P.klut_dom[tg.k0] || (uint32_t)xb >= P.klut_dom[tg.k1]) {
            fast_slow_2d(P, smem, t, xa, xb, cnt);
            continue;
        }
        if (agg && cnt > 1 && P.pairhh_off >= 0 && t == P.pair_t &&
            hh_add(smem + P.pairhh_off, P.pair_log2, ((uint64_t)(uint32_t)xa << 32) | (uint32_t)xb, cnt))
            continue;   // absorbed by the CTA's pair table (flushed once per distinct pair)
        const uint4 qa = swap ? b.e[NK - 1] : b.e[0], qb = swap ? b.e[0] : b.e[NK - 1];
        const uint32_t wm0 = tg.wmask0, wm1 = tg.wmask1, lw1 = tg.lw1, d = tg.d;
        // (r * w + b) & (w_m - 1) = b & (w_m - 1): the family's bucket at the matrix width
        if (tg.smem_off >= 0) {
            int32_t *row = sc + tg.smem_off;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (r >= (int)d) break;
                const uint32_t fa = lut_fld(qa, r), fb = lut_fld(qb, r);
                atomicAdd(row + ((((fa >> 1) & wm0) << lw1) | ((fb >> 1) & wm1)), ((fa ^ fb) & 1u) ? -cnt : cnt);
                row += tg.cells;
            }
        } else {
            int64_t *row = tg.counters;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (r >= (int)d) break;
                const uint32_t fa = lut_fld(qa, r), fb = lut_fld(qb, r);
                red_add_s64(row + ((((fa >> 1) & wm0) << lw1) | ((fb >> 1) & wm1)), ((fa ^ fb) & 1u) ? -cnt : cnt);
                row += tg.cells;
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
            SCAN_CHECK(!FULL || (pr[q].soff >= 0 && (r0 & 3) == 0));
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
        "@p8 cp.async.ca.shared.global" SCAN_L2HINT " [%0], [%1], 8;\n\t"
        "@!p8 cp.async.ca.shared.global" SCAN_L2HINT " [%0], [%1], 4;\n}" ::"r"(dst), "l"(src), "r"(is8)
        : "memory");
}
template <int W>
__device__ __forceinline__ void cp_async_fixed_if(bool on, uint32_t dst, const void *src) {
    if (W == 8)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                     "@p cp.async.ca.shared.global" SCAN_L2HINT " [%0], [%1], 8;\n}" ::"r"(dst), "l"(src), "r"((int)on)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                     "@p cp.async.ca.shared.global" SCAN_L2HINT " [%0], [%1], 4;\n}" ::"r"(dst), "l"(src), "r"((int)on)
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

// per-warp state of the lookup-table path (one pending batch, adaptive aggregation)
template <int NK>
struct FastState {
    Pend<NK> pend;
    bool agg;
    uint32_t actr;
};

template <int NK, bool FAST, bool T3>
__device__ __forceinline__ void drain_batch(const SParams &P, unsigned char *smem, const unsigned char *q,
                                            const uint32_t (&kbytes)[NK], uint32_t head, uint32_t n, FastState<NK> &fs) {
#ifdef SCAN_NOHASH   // timing experiments only (tools/build_variant.sh): results are wrong
    return;
#endif
    const int lane = threadIdx.x & 31;
    const bool valid = (uint32_t)lane < n;
    SCAN_CHECK(n <= 32);
    if (FAST) {   // int32 keys: load this batch's table entries, then apply the pending batch
        int32_t xr[NK];
        const unsigned char *e = q + ((head + lane) & (P.cap - 1)) * (NK * 8);
#pragma unroll
        for (int k = 0; k < NK; ++k) xr[k] = valid ? *reinterpret_cast<const int32_t *>(e + k * 8) : 0;
        Pend<NK> nw;
        fast_load<NK>(P, valid, xr, nw);
        process_fast<NK>(P, smem, fs.pend, fs.agg, fs.actr);
        fs.pend = nw;
        return;
    }
    uint64_t xk[NK];
    const unsigned char *e = q + ((head + lane) & (P.cap - 1)) * (NK * 8);
#pragma unroll
    for (int k = 0; k < NK; ++k)
        xk[k] = valid ? canon61(kbytes[k] == 8 ? *reinterpret_cast<const int64_t *>(e + k * 8)
                                               : (int64_t) * reinterpret_cast<const int32_t *>(e + k * 8))
                      : 0;
    process_batch<NK, T3>(P, smem, valid, xk);
}

// KW = 0: generic (any predicate kinds, key widths read at run time); KW = 4 / 8: every
// predicate is an int32 range and every key column is KW bytes wide (no kind or width
// branches; survivors' keys are gathered straight from the ballots).  T3: the hashing drain
// also serves 3-D tensor targets (KW = 0 instances, launched only when a tensor is present)
template <int NK, int NP, int KW, bool FAST, int SUB, bool T3>
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
        if (FAST && P.pairhh_off >= 0) {
            uint64_t *keys = reinterpret_cast<uint64_t *>(smem + P.pairhh_off);
            int *cnts = reinterpret_cast<int *>(smem + P.pairhh_off + (8u << P.pair_log2));
            for (uint32_t i = tid; i < (1u << P.pair_log2); i += kThreads) { keys[i] = kEmpty; cnts[i] = 0; }
        }
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
                    SCAN_CHECK(P.off_ring + ((grp + 1) * kStages) * P.stage_bytes <= P.off_kbuf);
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
    FastState<NK> fs;
    fs.pend.valid = false;
#pragma unroll
    for (int k = 0; k < NK; ++k) { fs.pend.e[k] = make_uint4(0, 0, 0, 0); fs.pend.x[k] = 0; }
    fs.agg = false;
    fs.actr = 0;
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t n_tiles = (uint32_t)P.n_tiles;
    constexpr int NPX = (NP > 0) ? NP : 1;
    uint32_t s = 0, ph = 0;
    for (uint32_t t = gid; t < n_tiles; t += G) {
        const uint64_t row0 = uint64_t(t) * (SUB * kTile);
        mbar_wait_a(full_a + s * 8, ph);
        const unsigned char *stage = smem + P.off_ring + (grp * kStages + s) * P.stage_bytes;
        const bool full_tile = t < P.n_full_tiles;   // staged by the producer
        if (NP > 0) {
          // a stage holds SUB sub-tiles of kTile rows (one column after another); each lane
          // evaluates 4 rows per sub-tile.  SUB > 1 only for predicates the host expects to be
          // very selective: one ballot then skips a sub-tile without survivors.
#pragma unroll 1
          for (int u = 0; u < SUB; ++u) {
            const int r0u = r0 + (int)u * kTile;
            bool m[4];
            if (full_tile) eval_preds<NPX, R32, true>(pr, stage, row0, r0u, 4, m);
            else {
                const int64_t rem = (int64_t)P.n_rows - (int64_t)(row0 + r0u);
                eval_preds<NPX, R32, false>(pr, stage, row0, r0u, rem <= 0 ? 0 : (rem >= 4 ? 4 : (int)rem), m);
            }
            if (SUB > 1) {
                // the ballot orders every lane's shared reads of stage s before lane 0 releases
                // it after the last sub-tile
                const uint32_t any = __ballot_sync(0xffffffffu, m[0] | m[1] | m[2] | m[3]);
                if (u + 1 == SUB && lane == 0) mbar_arrive_a(empty_a + s * 8);
                if (!any) continue;   // nothing appended: no cp.async group for this sub-tile
            }
            // one ballot per row slot; the ballots also order every lane's shared reads of
            // stage s before lane 0 releases it
            const uint32_t B0 = __ballot_sync(0xffffffffu, m[0]), B1 = __ballot_sync(0xffffffffu, m[1]);
            const uint32_t B2 = __ballot_sync(0xffffffffu, m[2]), B3 = __ballot_sync(0xffffffffu, m[3]);
            if (SUB == 1 && lane == 0) mbar_arrive_a(empty_a + s * 8);
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
                        kb[k] = reinterpret_cast<const unsigned char *>(kptr[k]) + (row0 + r0u) * (uint64_t)(KW ? KW : 8);
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
                    // list, in rounds that fit the ring (a sub-tile may hold more survivors than it)
                    if (m[0]) sts_u16(rl_a + 2 * __popc(B0 & lt), r0u);
                    if (m[1]) sts_u16(rl_a + 2 * (c0 + __popc(B1 & lt)), r0u + 1);
                    if (m[2]) sts_u16(rl_a + 2 * (c0 + c1 + __popc(B2 & lt)), r0u + 2);
                    if (m[3]) sts_u16(rl_a + 2 * (c0 + c1 + c2 + __popc(B3 & lt)), r0u + 3);
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
                                drain_batch<NK, FAST, T3>(P, smem, q, kbytes, head, n, fs);
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
            SCAN_CHECK(tail - head <= cap);
            // one cp.async group per sub-tile with survivors: wait_group kLag then guarantees
            // the entries appended kLag such sub-tiles ago have landed
            cp_commit();
            const uint32_t ready_end = tl[kLag - 1];
#pragma unroll
            for (int i = kLag - 1; i > 0; --i) tl[i] = tl[i - 1];
            tl[0] = tail;
            if (ready_end - head >= 32) {
                cp_wait_lag();
                __syncwarp();
                while (ready_end - head >= 32) { drain_batch<NK, FAST, T3>(P, smem, q, kbytes, head, 32, fs); head += 32; }
            }
          }
        } else {
            // keys are staged (no predicate): aggregate and update straight from the stage
            const int64_t rem = (int64_t)P.n_rows - (int64_t)(row0 + r0);
            const int valid = rem <= 0 ? 0 : (rem >= 4 ? 4 : (int)rem);
            const uint32_t bits = (1u << valid) - 1u;
            surv += __reduce_add_sync(0xffffffffu, (uint32_t)valid);
            uint64_t xs[4][NK];
            int32_t xraw[4][NK];   // FAST: the raw int32 keys (every key column is int32)
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
                    xraw[0][k] = v.x; xraw[1][k] = v.y; xraw[2][k] = v.z; xraw[3][k] = v.w;
                    xs[0][k] = canon61(v.x); xs[1][k] = canon61(v.y); xs[2][k] = canon61(v.z); xs[3][k] = canon61(v.w);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        int64_t v = 0;
                        if (full_tile) v = *reinterpret_cast<const int64_t *>(stage + ksoff[k] + (r0 + j) * 8);
                        else if (j < valid) v = __ldg(reinterpret_cast<const long long *>(kptr[k]) + row0 + r0 + j);
                        xs[j][k] = canon61(v);
                        xraw[j][k] = 0;   // never FAST (int64 key)
                    }
                }
            }
            if (FAST) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    Pend<NK> nw;
                    fast_load<NK>(P, (bits >> j) & 1u, xraw[j], nw);
                    process_fast<NK>(P, smem, fs.pend, fs.agg, fs.actr);
                    fs.pend = nw;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) process_batch<NK, T3>(P, smem, (bits >> j) & 1u, xs[j]);
            }
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
            drain_batch<NK, FAST, T3>(P, smem, q, kbytes, head, n, fs);
            head += n;
        }
    }

    if (FAST) process_fast<NK>(P, smem, fs.pend, fs.agg, fs.actr);   // the last pending batch
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
    // ---- flush the skewed-pair table of the L2-backed matrix (FAST): one table lookup per
    //      key and d counters per distinct pair, with the pair's count (linearity)
    if (FAST && P.pairhh_off >= 0) {
        const uint64_t *keys = reinterpret_cast<const uint64_t *>(smem + P.pairhh_off);
        const int *cnts = reinterpret_cast<const int *>(smem + P.pairhh_off + (8u << P.pair_log2));
        const STarget &tg = P.tgt[P.pair_t];
        for (uint32_t s = tid; s < (1u << P.pair_log2); s += kConsumers) {
            const uint64_t key = keys[s];
            const int c = cnts[s];
            if (key == kEmpty || c == 0) continue;
            const uint4 qa = __ldg(P.klut[tg.k0] + (uint32_t)(key >> 32)), qb = __ldg(P.klut[tg.k1] + (uint32_t)key);
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < (int)tg.d) {
                    const uint32_t fa = lut_fld(qa, r), fb = lut_fld(qb, r);
                    const uint32_t cell = (((fa >> 1) & tg.wmask0) << tg.lw1) | ((fb >> 1) & tg.wmask1);
                    red_add_s64(tg.counters + uint64_t(r) * tg.cells + cell, ((fa ^ fb) & 1u) ? -(int64_t)c : (int64_t)c);
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
    if (P.push.peers) {
        // fused merge: once every CTA's flush has landed (grid barrier of the cooperative
        // launch), the consumers of all CTAs push the table's partial slice to every rank
        consumer_sync();
        if (tid == 0) grid_arrive_wait(P.push_bar, gridDim.x);
        consumer_sync();
        peer_push_range(P.push, uint64_t(blockIdx.x) * kConsumers + tid, uint64_t(gridDim.x) * kConsumers);
    }
}

}  // namespace
