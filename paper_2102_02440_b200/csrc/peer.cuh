// peer.cuh — cross-GPU merge over peer memory (SURVEY.md §8(f) 4, P2P variant
// "partition, sketch, merge"): every rank adds its partial counters into every rank's merged
// buffer with red.add over NVLink (each process maps its peers' buffers with CUDA IPC), so
// when all ranks' pushes have completed every merged buffer holds the sum — integer addition,
// exact and order-independent.  Used as the tail of the fused scan (k_scan, after a grid-wide
// barrier: the transfer of one table's sketches starts as soon as its scan's last CTA is done,
// no NCCL kernel) and by the stand-alone k_peer_push.
#pragma once
#include <stdint.h>

namespace skb {

constexpr uint32_t kMaxPeers = 8;

struct PeerPush {
    const int64_t *src;             // this rank's partial slice (device)
    int64_t *dst[kMaxPeers];        // every rank's merged slice, as mapped in this process
    uint64_t n;                     // int64 elements
    uint32_t peers;                 // 0 = no push
    uint32_t owner_mode, rank;      // owner_mode: reduce-scatter (each element to its owner only)
    uint64_t offset, total;         // owner_mode: src's offset in, and the length of, the merged buffer
};

// first element of owner o's range (even, so a 16-byte pair never straddles two owners)
__host__ __device__ __forceinline__ uint64_t owner_lo(uint64_t total, uint32_t peers, uint32_t o) {
    return o >= peers ? total : ((total * o / peers) & ~uint64_t(1));
}
__device__ __forceinline__ uint32_t owner_of(uint64_t e, uint64_t total, uint32_t peers) {
    const uint64_t g = e * peers / (total ? total : 1);
    uint32_t o = (uint32_t)(g < peers - 1 ? g : peers - 1);
    while (o > 0 && e < owner_lo(total, peers, o)) --o;
    while (o + 1 < peers && e >= owner_lo(total, peers, o + 1)) ++o;
    return o;
}

// red.add of one int64 into a (possibly peer) global address; the u64 add is the s64 add in
// two's complement
__device__ __forceinline__ void peer_red_s64(int64_t *p, int64_t v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)v) : "memory");
}

// thread `idx` of `stride` pushes elements idx*2, idx*2+1, (idx+stride)*2, ... of the slice
// (16-byte loads that bypass L1: the partial was written by L2 atomics); zero counters are
// skipped (no traffic)
__device__ __forceinline__ void peer_push_range(const PeerPush &pp, uint64_t idx, uint64_t stride) {
    const uint64_t pairs = pp.n >> 1;
    const longlong2 *s2 = reinterpret_cast<const longlong2 *>(pp.src);
    for (uint64_t e = idx; e < pairs; e += stride) {
        const longlong2 v = __ldcg(s2 + e);
        if (!(v.x | v.y)) continue;
        if (pp.owner_mode) {
            const uint32_t o = owner_of(pp.offset + 2 * e, pp.total, pp.peers);
            if (v.x) peer_red_s64(pp.dst[o] + 2 * e, v.x);
            if (v.y) peer_red_s64(pp.dst[o] + 2 * e + 1, v.y);
            continue;
        }
        if (v.x)
            for (uint32_t p = 0; p < pp.peers; ++p) peer_red_s64(pp.dst[p] + 2 * e, v.x);
        if (v.y)
            for (uint32_t p = 0; p < pp.peers; ++p) peer_red_s64(pp.dst[p] + 2 * e + 1, v.y);
    }
    if ((pp.n & 1) && idx == 0) {
        const int64_t v = __ldcg(reinterpret_cast<const long long *>(pp.src) + pp.n - 1);
        if (v && pp.owner_mode) peer_red_s64(pp.dst[owner_of(pp.offset + pp.n - 1, pp.total, pp.peers)] + pp.n - 1, v);
        else if (v)
            for (uint32_t p = 0; p < pp.peers; ++p) peer_red_s64(pp.dst[p] + pp.n - 1, v);
    }
}

// one-shot grid barrier of a cooperative launch (every CTA co-resident): called by one thread
// per CTA; *bar starts at 0
__device__ __forceinline__ void grid_arrive_wait(unsigned int *bar, unsigned int n_ctas) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        if (v >= n_ctas) break;
        __nanosleep(100);
    }
}

}  // namespace skb
