// scan.cuh — host-side description of one fused-scan call (shared by update.cu and scan.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "compass_b200.h"
#include "peer.cuh"

namespace skb {

struct ScanCall {
    uint32_t n_cols = 0;
    const void *col_ptr[16];
    uint32_t col_bytes[16];
    uint64_t col_domain[16];    // key-domain hints (0 = unknown)
    uint64_t n_rows = 0;
    uint32_t n_preds = 0;
    uint32_t pred_col[8], pred_kind[8];
    int64_t pred_lo[8], pred_hi[8];
    const int64_t *pred_set[8];
    uint32_t pred_n[8];
    uint32_t n_targets = 0;
    int64_t *tgt_counters[16];
    uint32_t tgt_ndim[16], tgt_d[16], tgt_w[16][3], tgt_key[16][3];
    const uint64_t *tgt_seeds[16];
    const uint64_t *tgt_seeds_host[16];   // host copies [ndim][d][6] (hash-unit sharing)
    sk_sketch *tgt_sketch[16];             // target handles (per-sketch hash lookup tables)
    unsigned long long *survivors = nullptr;
    PeerPush push{};                       // cross-GPU merge over peer memory (peers = 0: none)
};

// Launch the optimised persistent scan if the call fits its envelope (sets *launched); with
// c.push.peers, *pushed says whether the push was fused into the scan (else the caller runs
// peer_push_launch after it).
sk_status scan_launch(const ScanCall &c, cudaStream_t stream, bool *launched, bool *pushed);

// Stand-alone push of a partial slice into every rank's merged slice (peer.cuh).
sk_status peer_push_launch(const PeerPush &pp, cudaStream_t stream);
// Owner-mode merge, second half: copy the other owners' ranges into this rank's buffer.
sk_status peer_gather_launch(const PeerPush &pp, cudaStream_t stream);

}  // namespace skb
