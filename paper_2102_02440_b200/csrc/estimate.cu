// estimate.cu — sketch composition: two-way and multi-way join estimates
// (PAPER.md:197-201 two-way; PAPER.md:221-225 partitioned; PAPER.md:234-240
// merging) and the greedy enumerator.
//
// Exactness.  E_r is an integer (a sum of products of integer counters), computed
// exactly by one of three engines: (1) two-way sub-plans, an int128 dot product per row
// (k_dot128; rows not provably inside int128 are flagged and redone by (3)); (2) matrix-
// free multi-way sub-plans whose rigorous bound (message-passing node bounds from the
// survivor counts, re-verified with L1 norms measured on the device) is <= 2^125, an
// int128 (or int64, when a node's bound is <= 2^61) message-passing engine; (3) every
// other sub-plan, modulo K primes below 2^26 (Barrett reduction, kMods), K chosen from the
// same bound, reconstructed on the host by Garner's mixed-radix CRT.  The host takes the
// median over rows and rounds it once to fp64 (round-to-nearest-even).
//
// Contraction.  The sub-plan's tensor network is contracted by message passing
// over a spanning tree rooted at the lowest-index table; a single cycle is
// handled by conditioning one cycle edge on each of its buckets (batched).
// Node kinds: 1-D sketch, built matrix, min-abs merged view (<= 3 legs).  A
// merged node contracts its first child leg with the identity of SURVEY.md O9:
// with |c| sorted ascending and prefix sums P1 = sum x, P2 = sum x*c,
//   sum_i x_i fold(L, c_i, R) = m(L,R) * sum_{|c_i|>=|L|} x_i
//                             + sum_{|c_i|<|L|, |c_i|<=|R|} x_i c_i
//                             + R * sum_{|R|<|c_i|<|L|} x_i.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <deque>
#include <set>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace skb;

namespace {

constexpr int kMaxMod = 28;
// the 28 largest primes below 2^26 (pinned by tests/test_abi.py): residue products fit in
// 52 bits, so up to 4096 of them accumulate exactly in one 64-bit register
const uint32_t kPrimes[kMaxMod] = {67108859, 67108837, 67108819, 67108777, 67108763, 67108757, 67108753,
                                   67108747, 67108739, 67108729, 67108721, 67108709, 67108693, 67108669,
                                   67108667, 67108661, 67108649, 67108633, 67108597, 67108579, 67108529,
                                   67108511, 67108507, 67108493, 67108471, 67108463, 67108453, 67108439};
enum { KV = 0, KM = 1, KG = 2, KT = 3 };  // vector, matrix, merged, 3-D tensor
enum { RCHILD = 0, RPARENT = 1, RFIXED = 2 };

struct Mods {
    int K;
    uint64_t m[kMaxMod];    // primes < 2^26
    uint64_t mu[kMaxMod];   // floor(2^64 / m) (Barrett)
};

// ---------------------------------------------------------------- device modular arithmetic
// t < 2^64 -> t mod m (Barrett: q >= t/m - 2, so at most two corrections)
__device__ __forceinline__ uint64_t mm_red(uint64_t t, uint64_t m, uint64_t mu) {
    const uint64_t q = __umul64hi(t, mu);
    uint64_t r = t - q * m;
    if (r >= m) r -= m;
    if (r >= m) r -= m;
    return r;
}
__device__ __forceinline__ uint64_t mm_mul(uint64_t x, uint64_t y, uint64_t m, uint64_t mu) {
    return mm_red(x * y, m, mu);
}
__device__ __forceinline__ uint64_t mm_add(uint64_t x, uint64_t y, uint64_t m) {
    const uint64_t s = x + y;
    return s >= m ? s - m : s;
}
__device__ __forceinline__ uint64_t mm_sub(uint64_t x, uint64_t y, uint64_t m) {
    return x >= y ? x - y : x + (m - y);
}
__device__ __forceinline__ uint64_t uabs(int64_t v) { return v < 0 ? (uint64_t)(-(v + 1)) + 1ULL : (uint64_t)v; }
__device__ __forceinline__ uint64_t mm_i64(int64_t v, uint64_t m, uint64_t mu) {
    const uint64_t r = mm_red(uabs(v), m, mu);
    return (v < 0 && r) ? m - r : r;
}

// ---------------------------------------------------------------- small kernels
// per (item, row): sum |v| over `cells` counters (blockIdx.z = chunk; atomically accumulated).
// Saturating: a row whose L1 reaches 2^64 (caller-owned counters can hold any int64) reads
// UINT64_MAX, which the host takes as the worst case 2^63 * cells (the bound stays rigorous).
__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
    const unsigned long long c = a + b;
    return c < a ? ~0ULL : c;
}
struct L1Item { const int64_t *p; uint32_t d; uint32_t cells; };
constexpr int kMaxL1Items = 48;
struct L1Items { L1Item it[kMaxL1Items]; int n; };
__global__ void k_l1(const __grid_constant__ L1Items items, unsigned long long *out, int maxd) {
    const L1Item it = items.it[blockIdx.x];
    const uint32_t r = blockIdx.y;
    if (r >= it.d) return;
    const uint32_t chunk = (it.cells + gridDim.z - 1) / gridDim.z;
    const uint32_t c0 = blockIdx.z * chunk, c1 = min(it.cells, c0 + chunk);
    unsigned long long s = 0;
    for (uint32_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) s = sat_add(s, uabs(it.p[uint64_t(r) * it.cells + i]));
    __shared__ unsigned long long red[32];
    for (int o = 16; o > 0; o >>= 1) s = sat_add(s, __shfl_xor_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = sat_add(t, red[i]);
        if (t) {
            unsigned long long *p = &out[blockIdx.x * maxd + r];
            unsigned long long old = *p, seen;
            while ((seen = atomicCAS(p, old, sat_add(old, t))) != old) old = seen;
        }
    }
}

// fold [d][wn0][wn1] -> [d][w0][w1]: out[r][i][j] = sum_{s,t} in[r][i + s w0][j + t w1]  (O5)
__global__ void k_fold(const int64_t *in, int64_t *out, uint32_t d, uint32_t wn0, uint32_t wn1, uint32_t w0, uint32_t w1) {
    const uint64_t total = uint64_t(d) * w0 * w1;
    for (uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < total; o += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t j = (uint32_t)(o % w1);
        const uint32_t i = (uint32_t)((o / w1) % w0);
        const uint32_t r = (uint32_t)(o / (uint64_t(w0) * w1));
        int64_t s = 0;
        for (uint32_t a = i; a < wn0; a += w0)
            for (uint32_t b = j; b < wn1; b += w1) s += in[(uint64_t(r) * wn0 + a) * wn1 + b];
        out[o] = s;
    }
}

// fold [d][wn0][wn1][wn2] -> [d][w0][w1][w2] along every axis (O5 per dimension)
__global__ void k_fold3(const int64_t *in, int64_t *out, uint32_t d, uint32_t wn0, uint32_t wn1, uint32_t wn2, uint32_t w0,
                        uint32_t w1, uint32_t w2) {
    const uint64_t total = uint64_t(d) * w0 * w1 * w2;
    for (uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < total; o += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t k = (uint32_t)(o % w2);
        const uint32_t j = (uint32_t)((o / w2) % w1);
        const uint32_t i = (uint32_t)((o / (uint64_t(w1) * w2)) % w0);
        const uint32_t r = (uint32_t)(o / (uint64_t(w0) * w1 * w2));
        int64_t s = 0;
        for (uint32_t a = i; a < wn0; a += w0)
            for (uint32_t b = j; b < wn1; b += w1)
                for (uint32_t c = k; c < wn2; c += w2) s += in[((uint64_t(r) * wn0 + a) * wn1 + b) * wn2 + c];
        out[o] = s;
    }
}

// per row: sort indices by |c| ascending (bitonic, w a power of two, w <= 8192)
__global__ void k_sort_abs(const int64_t *c, uint32_t w, int32_t *ord, uint64_t *sabs, int32_t *rank, int64_t *csorted) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *key = reinterpret_cast<uint64_t *>(sm);
    uint32_t *idx = reinterpret_cast<uint32_t *>(key + w);
    const uint32_t r = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
        key[i] = uabs(c[uint64_t(r) * w + i]);
        idx[i] = i;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= w; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = key[i] > key[l] || (key[i] == key[l] && idx[i] > idx[l]);
                    if (gt == up) {
                        uint64_t tk = key[i]; key[i] = key[l]; key[l] = tk;
                        uint32_t ti = idx[i]; idx[i] = idx[l]; idx[l] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
        ord[uint64_t(r) * w + i] = (int32_t)idx[i];
        sabs[uint64_t(r) * w + i] = key[i];
        rank[uint64_t(r) * w + idx[i]] = (int32_t)i;
        csorted[uint64_t(r) * w + i] = c[uint64_t(r) * w + idx[i]];
    }
}

// ---------------------------------------------------------------- node kernels
struct Node {
    int kind, nl;
    int role[3];
    int w[3];
    const int64_t *data[3];     // folded; VEC [d][w0]; MAT [d][w0][w1]; MERGED data[q] = [d][w_q]
    const uint64_t *msg[3];     // child messages, layout [K][d][bm][w]
    int bm[3];
    int qc;                     // merged: contracted child leg
    const int32_t *ord;         // merged: [d][w_qc]
    const uint64_t *sabs;       // merged: [d][w_qc]
    const int64_t *csorted;     // merged: constituent qc in |c|-sorted order [d][w_qc]
    const int32_t *out_perm;    // parent message written at out_perm[r][o] (the parent's sorted order), or null
    const uint32_t *rank[3];    // merged: per other leg q, [d][w_q] = #{|c| < |v|} | #{|c| <= |v|} << 16 of
                                // its constituent values v against the contracted leg's sorted |c| (or null)
    uint64_t *out;              // parent message [K][d][out_bm][w_p], or root partials [K][d][B][tiles]
    int out_bm;
    int m64;                    // exact engine: bit q = leg q's child message is stored as int64
    int out64;                  // exact engine: this node's parent message is stored as int64
    int B, tiles, d;
    int64_t b0;
};

__device__ __forceinline__ const uint64_t *msg_row(const Node &n, int q, int k, int r, int bb, int Kd_unused) {
    const int bm = n.bm[q];
    return n.msg[q] + ((uint64_t(k) * n.d + r) * bm + (bm > 1 ? bb : 0)) * (uint64_t)n.w[q];
}

__device__ __forceinline__ uint64_t block_sum_mod(uint64_t v, uint64_t m, uint64_t *red) {
    // warp
    for (int o = 16; o > 0; o >>= 1) v = mm_add(v, __shfl_xor_sync(0xffffffffu, v, o), m);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    uint64_t t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = mm_add(t, red[i], m);
    return t;
}

// value of a node's tensor at per-leg indices (merged: left fold of the min-abs rule)
__device__ __forceinline__ int64_t tensor_val(const Node &n, int r, const int64_t *idx) {
    if (n.kind == KV) return n.data[0][uint64_t(r) * n.w[0] + idx[0]];
    if (n.kind == KM) return n.data[0][(uint64_t(r) * n.w[0] + idx[0]) * n.w[1] + idx[1]];
    if (n.kind == KT) return n.data[0][((uint64_t(r) * n.w[0] + idx[0]) * n.w[1] + idx[1]) * n.w[2] + idx[2]];
    int64_t acc = n.data[0][uint64_t(r) * n.w[0] + idx[0]];
    for (int q = 1; q < n.nl; ++q) {
        const int64_t v = n.data[q][uint64_t(r) * n.w[q] + idx[q]];
        if (!(uabs(acc) <= uabs(v))) acc = v;
    }
    return acc;
}

// VEC / MAT node, or a merged leaf.  blockIdx.x = (k*d + r)*B + bb, blockIdx.y = tile of the outer index.
__global__ void k_node_dense(const __grid_constant__ Node n, const __grid_constant__ Mods md) {
    __shared__ uint64_t red[32];
    const int B = n.B;
    const int bb = blockIdx.x % B;
    const int r = (blockIdx.x / B) % n.d;
    const int k = blockIdx.x / (B * n.d);
    const uint64_t mu = md.mu[k];
    const uint64_t m = md.m[k];
    const int64_t b = n.b0 + bb;
    int qp = -1, qf = -1, qc0 = -1, qc1 = -1, qc2 = -1;
    for (int q = 0; q < n.nl; ++q) {
        if (n.role[q] == RPARENT) qp = q;
        else if (n.role[q] == RFIXED) qf = q;
        else if (qc0 < 0) qc0 = q;
        else if (qc1 < 0) qc1 = q;
        else qc2 = q;
    }
    // outer leg: parent if any, else first child; inner legs: the (other) children, a second
    // one only for a 3-D tensor with three free legs
    const int qo = qp >= 0 ? qp : qc0;
    const int qi = qp >= 0 ? qc0 : qc1;
    const int qj = qp >= 0 ? qc1 : qc2;
    const int wo = qo >= 0 ? n.w[qo] : 1;
    const int wi = qi >= 0 ? n.w[qi] : 1;
    const int wj = qj >= 0 ? n.w[qj] : 1;
    const uint64_t *xo = (qo >= 0 && n.role[qo] == RCHILD) ? msg_row(n, qo, k, r, bb, 0) : nullptr;
    const uint64_t *xi = (qi >= 0) ? msg_row(n, qi, k, r, bb, 0) : nullptr;
    const uint64_t *xj = (qj >= 0) ? msg_row(n, qj, k, r, bb, 0) : nullptr;
    uint64_t acc = 0;
    const int per_tile = (wo + n.tiles - 1) / n.tiles;
    const int o_begin = blockIdx.y * per_tile, o_end = min(wo, o_begin + per_tile);
    for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
        uint64_t s = 0;
        for (int i = 0; i < wi; ++i) {
            for (int j = 0; j < wj; ++j) {
                int64_t idx[3] = {0, 0, 0};
                if (qo >= 0) idx[qo] = o;
                if (qi >= 0) idx[qi] = i;
                if (qj >= 0) idx[qj] = j;
                if (qf >= 0) idx[qf] = b;
                uint64_t term = mm_i64(tensor_val(n, r, idx), m, mu);
                if (xi) term = mm_mul(term, xi[i], m, mu);
                if (xj) term = mm_mul(term, xj[j], m, mu);
                s = mm_add(s, term, m);
            }
        }
        if (qp >= 0) {
            const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
            n.out[((uint64_t(k) * n.d + r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo] = s;
        } else {
            if (xo) s = mm_mul(s, xo[o], m, mu);
            acc = mm_add(acc, s, m);
        }
    }
    if (qp < 0) {
        const uint64_t t = block_sum_mod(acc, m, red);
        if (threadIdx.x == 0) n.out[((uint64_t(k) * n.d + r) * B + bb) * n.tiles + blockIdx.y] = t;
    }
}

// merged node (min-abs view over <= 3 constituents), first child leg contracted by O9.
// One CTA per (row r, conditioned bucket bb, tile of the outer leg) handles all K moduli:
// the |c|-threshold positions of each outer index (binary searches, independent of the
// modulus) are computed once into shared memory, then per modulus only the prefix sums
// of the message and one O(1) combination per output remain.
__device__ __forceinline__ void merged_LR(const Node &n, int r, int qc, int qf, int qo, int qi, int64_t b, int o, int i,
                                          bool &hasL, int64_t &L, bool &hasR, int64_t &R) {
    hasL = hasR = false;
    L = R = 0;
    for (int q = 0; q < n.nl; ++q) {
        if (q == qc) continue;
        const int64_t ix = (q == qf) ? b : (q == qo ? o : i);
        const int64_t v = n.data[q][uint64_t(r) * n.w[q] + ix];
        if (q < qc) { if (!hasL || !(uabs(L) <= uabs(v))) L = v; hasL = true; }
        else { if (!hasR || !(uabs(R) <= uabs(v))) R = v; hasR = true; }
    }
}

// #{s : S[s] < t} and #{s : S[s] <= t} over the ascending array S[0..w)
__device__ __forceinline__ int count_lt(const uint64_t *S, int w, uint64_t t) {
    int lo = 0, hi = w;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (S[mid] < t) lo = mid + 1; else hi = mid; }
    return lo;
}
__device__ __forceinline__ int count_le(const uint64_t *S, int w, uint64_t t) {
    int lo = 0, hi = w;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (S[mid] <= t) lo = mid + 1; else hi = mid; }
    return lo;
}

// L, R and their threshold positions in the contracted leg's sorted |c|: from the per-leg rank
// tables when present (L and R are each one constituent value, so its precomputed ranks are
// the thresholds; two independent loads), else by binary search over S
__device__ __forceinline__ void merged_thr(const Node &n, int r, int qc, int qf, int qo, int qi, int64_t b, int o, int i,
                                           const uint64_t *S, int wq, bool &hasL, int64_t &L, bool &hasR, int64_t &R,
                                           int &nless, int &nle) {
    hasL = hasR = false;
    L = R = 0;
    int qL = -1, qR = -1;
    int64_t xL = 0, xR = 0;
    for (int q = 0; q < n.nl; ++q) {
        if (q == qc) continue;
        const int64_t ix = (q == qf) ? b : (q == qo ? o : i);
        const int64_t v = n.data[q][uint64_t(r) * n.w[q] + ix];
        if (q < qc) { if (!hasL || !(uabs(L) <= uabs(v))) { L = v; qL = q; xL = ix; } hasL = true; }
        else { if (!hasR || !(uabs(R) <= uabs(v))) { R = v; qR = q; xR = ix; } hasR = true; }
    }
    if (n.rank[0] || n.rank[1] || n.rank[2]) {
        nless = hasL ? (int)(n.rank[qL][uint64_t(r) * n.w[qL] + xL] & 0xffffu) : 0;
        nle = hasR ? (int)(n.rank[qR][uint64_t(r) * n.w[qR] + xR] >> 16) : 0;
    } else {
        nless = hasL ? count_lt(S, wq, uabs(L)) : 0;
        nle = hasR ? count_le(S, wq, uabs(R)) : 0;
    }
}

// per row and every other leg q of a merged node: the ranks of its constituent values in the
// contracted leg's sorted |c| (computed once per node, shared by every conditioned bucket,
// every outer index and every modulus).  out[q] = [d][w_q]
__global__ void k_merged_rank(const __grid_constant__ Node n, uint32_t *out0, uint32_t *out1, uint32_t *out2) {
    const int r = blockIdx.y;
    const int wq = n.w[n.qc];
    const uint64_t *S = n.sabs + uint64_t(r) * wq;
    uint32_t *outs[3] = {out0, out1, out2};
    for (int q = 0; q < n.nl; ++q) {
        if (q == n.qc || !outs[q]) continue;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n.w[q]; i += gridDim.x * blockDim.x) {
            const uint64_t v = uabs(n.data[q][uint64_t(r) * n.w[q] + i]);
            outs[q][uint64_t(r) * n.w[q] + i] = (uint32_t)count_lt(S, wq, v) | ((uint32_t)count_le(S, wq, v) << 16);
        }
    }
}

// sum_i x_i fold(L, c_i, R) mod m from the prefix sums P1 (x) and P2 (x*c)
__device__ __forceinline__ uint64_t o9_value(const uint64_t *P1, const uint64_t *P2, int wq, bool hasL, int64_t L,
                                             bool hasR, int64_t R, int nless, int nle, uint64_t m, uint64_t mu) {
    uint64_t V;
    if (hasL) {
        const int64_t win = (hasR && !(uabs(L) <= uabs(R))) ? R : L;
        V = mm_mul(mm_i64(win, m, mu), mm_sub(P1[wq], P1[nless], m), m, mu);
        int endB = nless;
        if (hasR && nle < endB) {
            V = mm_add(V, mm_mul(mm_i64(R, m, mu), mm_sub(P1[endB], P1[nle], m), m, mu), m);
            endB = nle;
        }
        V = mm_add(V, P2[endB], m);
    } else {
        V = mm_add(mm_mul(mm_i64(R, m, mu), mm_sub(P1[wq], P1[nle], m), m, mu), P2[nle], m);
    }
    return V;
}

// Matrix node with one child leg and one parent leg, batched over the conditioned bucket:
// out[b][j] = sum_i x[b][i] * M(i, j) mod m — a modular GEMM.  Residues are < 2^26, so
// products (< 2^52) accumulate exactly in 64 bits (IMAD.WIDE.U32) for 4096 steps between
// Barrett reductions.  Tile 32 b x 64 j x 32 i, 8 outputs per thread.
constexpr int GBM = 32, GBN = 64, GBK = 32;
__global__ void __launch_bounds__(256) k_node_mat_gemm(const __grid_constant__ Node n, const __grid_constant__ Mods md, int qc,
                                                       const uint32_t *Rc) {
    __shared__ uint32_t Xs[GBK][GBM + 1];
    __shared__ uint32_t Ms[GBK][GBN + 4];
    const int k = blockIdx.x / n.d, r = blockIdx.x % n.d;
    const uint64_t m = md.m[k], mu = md.mu[k];
    const int nbt = (n.B + GBM - 1) / GBM;
    const int b0 = (blockIdx.y % nbt) * GBM, j0 = (blockIdx.y / nbt) * GBN;
    const int qp = 1 - qc;
    const int wi = n.w[qc], wj = n.w[qp];
    const int64_t *T = n.data[0] + uint64_t(r) * n.w[0] * n.w[1];
    const int tid = threadIdx.x;
    const int tb = (tid >> 4) * 2, tj = (tid & 15) * 4;
    uint64_t acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    int since = 0;
    for (int i0 = 0; i0 < wi; i0 += GBK) {
        for (int e = tid; e < GBK * GBM; e += 256) {
            const int ii = e % GBK, bl = e / GBK;
            const int b = b0 + bl, i = i0 + ii;
            Xs[ii][bl] = (b < n.B && i < wi) ? (uint32_t)msg_row(n, qc, k, r, b, 0)[i] : 0u;
        }
        if (Rc) {   // residues of this matrix in this orientation, precomputed once per batch
            const uint32_t *R = Rc + (uint64_t(k) * n.d + r) * (uint64_t(wi) * wj);
            for (int e = tid; e < GBK * GBN; e += 256) {
                const int jj = e % GBN, ii = e / GBN;
                const int i = i0 + ii, j = j0 + jj;
                Ms[ii][jj] = (i < wi && j < wj) ? __ldg(R + uint64_t(i) * wj + j) : 0u;
            }
        } else
        for (int e = tid; e < GBK * GBN; e += 256) {
            int ii, jj;
            if (qc == 0) { jj = e % GBN; ii = e / GBN; } else { ii = e % GBK; jj = e / GBK; }
            const int i = i0 + ii, j = j0 + jj;
            uint32_t v = 0;
            if (i < wi && j < wj) v = (uint32_t)mm_i64(qc == 0 ? T[uint64_t(i) * wj + j] : T[uint64_t(j) * wi + i], m, mu);
            Ms[ii][jj] = v;
        }
        __syncthreads();
#pragma unroll 8
        for (int ii = 0; ii < GBK; ++ii) {
            const uint64_t x0 = Xs[ii][tb], x1 = Xs[ii][tb + 1];
            const uint64_t m0 = Ms[ii][tj], m1 = Ms[ii][tj + 1], m2 = Ms[ii][tj + 2], m3 = Ms[ii][tj + 3];
            acc[0][0] += x0 * m0; acc[0][1] += x0 * m1; acc[0][2] += x0 * m2; acc[0][3] += x0 * m3;
            acc[1][0] += x1 * m0; acc[1][1] += x1 * m1; acc[1][2] += x1 * m2; acc[1][3] += x1 * m3;
        }
        __syncthreads();
        since += GBK;
        if (since >= 4096) {
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[a][c] = mm_red(acc[a][c], m, mu);
            since = 0;
        }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const int b = b0 + tb + a;
        if (b >= n.B) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = j0 + tj + c;
            if (j >= wj) continue;
            const int jo = n.out_perm ? n.out_perm[uint64_t(r) * wj + j] : j;
            n.out[((uint64_t(k) * n.d + r) * n.out_bm + (n.out_bm > 1 ? b : 0)) * wj + jo] = mm_red(acc[a][c], m, mu);
        }
    }
}

// ---------------------------------------------------------------- tensor-core modular GEMM
// The same product as k_node_mat_gemm, out[b][j] = sum_i x[b][i] M(i, j) mod m, on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM).  Residues
// (< 2^26) are split into 4 byte planes, x = sum_a 2^(8a) x_a and M = sum_c 2^(8c) M_c; the
// 16 byte-plane products with a + c = s accumulate in one of 7 int32 TMEM accumulators
// D_s (every entry <= 4 * w_i * 255^2 < 2^31 for w_i <= 8192, exact), and the epilogue forms
// sum_s D_s * (2^(8s) mod m) (< 2^60) and reduces it once.  The result is the same integer
// residue as the CUDA-core kernel's, by construction.
//
// CTA tile 128 b x 64 j, k-blocks of 64 i; 3-stage smem ring of byte planes (A: 4 x 128 x
// 64 B, B: 4 x 64 x 64 B) filled by all 256 threads (residues -> bytes, canonical K-major
// no-swizzle core-matrix layout: 8 rows x 16 B per core matrix, SBO = 128 B between 8-row
// groups, LBO = rows x 16 B between 16-byte K chunks), one elected thread issues the 32
// MMAs (128 x 64 x 32) of a stage and commits them to the stage's mbarrier; 512 TMEM
// columns (7 x 64 used), one CTA per SM.
constexpr int TC_M = 128, TC_N = 64, TC_KB = 64, TC_ST = 3;
constexpr int TC_A_PLANE = TC_M * TC_KB, TC_B_PLANE = TC_N * TC_KB;          // bytes
constexpr int TC_STAGE = 4 * TC_A_PLANE + 4 * TC_B_PLANE;                    // 48 KB
constexpr int TC_SMEM = TC_ST * TC_STAGE + 64;                               // + barriers, TMEM slot

__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SM100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4
    // [32,46), version 1 [46,48), base offset 0, layout SWIZZLE_NONE (0) [61,64)
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tc_mbar_wait(uint32_t a, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(a),
                 "r"(ph) : "memory");
}

__global__ void __launch_bounds__(256, 1) k_node_mat_gemm_tc(const __grid_constant__ Node n, const __grid_constant__ Mods md,
                                                             int qc, const uint32_t *Rc) {
    extern __shared__ __align__(1024) unsigned char tsm[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tsm);
    const uint32_t bar0 = sbase + TC_ST * TC_STAGE;     // TC_ST mbarriers, then the TMEM address slot
    const uint32_t slot = bar0 + 8 * TC_ST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int k = blockIdx.x / n.d, r = blockIdx.x % n.d;
    const uint64_t m = md.m[k], mu = md.mu[k];
    const int nbt = (n.B + TC_M - 1) / TC_M;
    const int b0 = (blockIdx.y % nbt) * TC_M, j0 = (blockIdx.y / nbt) * TC_N;
    const int qp = 1 - qc;
    const int wi = n.w[qc], wj = n.w[qp];
    const uint32_t *R = Rc + (uint64_t(k) * n.d + r) * (uint64_t(wi) * wj);

    if (tid == 0) {
        for (int s = 0; s < TC_ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(slot) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t tmem;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(slot) : "memory");

    // instruction descriptor: D s32 [4,6) = 2, A/B u8, K-major, N >> 3 at [17,23), M >> 4 at [24,29)
    const uint32_t idesc = (2u << 4) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
    const int nkb = (wi + TC_KB - 1) / TC_KB;
    for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % TC_ST;
        if (kb >= TC_ST) tc_mbar_wait(bar0 + 8 * st, (uint32_t)((kb / TC_ST - 1) & 1));   // MMAs of kb - TC_ST done
        unsigned char *A = tsm + st * TC_STAGE, *Bp = A + 4 * TC_A_PLANE;
        const int i0 = kb * TC_KB;
        // A: 128 rows x 4 chunks of 16 i; one item = 16 residues of one row -> 16 B per plane
        for (int e = tid; e < TC_M * 4; e += 256) {
            const int row = e % TC_M, c = e / TC_M;
            const int b = b0 + row, ib = i0 + c * 16;
            uint32_t w[4][4];
            if (b < n.B && ib + 16 <= wi) {
                const uint64_t *x = msg_row(n, qc, k, r, b, 0) + ib;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t v[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) v[t] = (uint32_t)__ldg(reinterpret_cast<const unsigned long long *>(x) + q * 4 + t);
#pragma unroll
                    for (int a = 0; a < 4; ++a)
                        w[a][q] = ((v[0] >> (8 * a)) & 0xFF) | (((v[1] >> (8 * a)) & 0xFF) << 8) |
                                  (((v[2] >> (8 * a)) & 0xFF) << 16) | (((v[3] >> (8 * a)) & 0xFF) << 24);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t v[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int i = ib + q * 4 + t;
                        v[t] = (b < n.B && i < wi) ? (uint32_t)msg_row(n, qc, k, r, b, 0)[i] : 0u;
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
                        w[a][q] = ((v[0] >> (8 * a)) & 0xFF) | (((v[1] >> (8 * a)) & 0xFF) << 8) |
                                  (((v[2] >> (8 * a)) & 0xFF) << 16) | (((v[3] >> (8 * a)) & 0xFF) << 24);
                }
            }
            const int off = c * (TC_M * 16) + (row >> 3) * 128 + (row & 7) * 16;
#pragma unroll
            for (int a = 0; a < 4; ++a)
                *reinterpret_cast<uint4 *>(A + a * TC_A_PLANE + off) = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
        }
        // B (K-major: row j holds M(i, j) for the 64 i of the block): 64 rows x 4 chunks
        for (int e = tid; e < TC_N * 4; e += 256) {
            const int jr = e % TC_N, c = e / TC_N;
            const int j = j0 + jr, ib = i0 + c * 16;
            uint32_t w[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int i = ib + q * 4 + t;
                    v[t] = (j < wj && i < wi) ? __ldg(R + uint64_t(i) * wj + j) : 0u;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
                    w[a][q] = ((v[0] >> (8 * a)) & 0xFF) | (((v[1] >> (8 * a)) & 0xFF) << 8) |
                              (((v[2] >> (8 * a)) & 0xFF) << 16) | (((v[3] >> (8 * a)) & 0xFF) << 24);
            }
            const int off = c * (TC_N * 16) + (jr >> 3) * 128 + (jr & 7) * 16;
#pragma unroll
            for (int a = 0; a < 4; ++a)
                *reinterpret_cast<uint4 *>(Bp + a * TC_B_PLANE + off) = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a_s = sbase + st * TC_STAGE, b_s = a_s + 4 * TC_A_PLANE;
            for (int a = 0; a < 4; ++a)
                for (int c = 0; c < 4; ++c) {
                    const int s = a + c;
                    const uint32_t dt = tmem + (uint32_t)(s * TC_N);
                    for (int ks = 0; ks < TC_KB / 32; ++ks) {
                        // first write of D_s: (kb, ks) == (0, 0) and the first (a, c) with a + c = s
                        const bool first = kb == 0 && ks == 0 && (s <= 3 ? a == 0 : c == 3);
                        const uint64_t ad = tc_sdesc(a_s + a * TC_A_PLANE + ks * 2 * (TC_M * 16), TC_M * 16, 128);
                        const uint64_t bd = tc_sdesc(b_s + c * TC_B_PLANE + ks * 2 * (TC_N * 16), TC_N * 16, 128);
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                                     "l"(ad), "l"(bd), "r"(idesc), "r"(first ? 0u : 1u) : "memory");
                    }
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar0 + 8 * st)
                         : "memory");
        }
    }
    // the last commit covers every MMA issued before it
    {
        const int st = (nkb - 1) % TC_ST;
        tc_mbar_wait(bar0 + 8 * st, (uint32_t)(((nkb - 1) / TC_ST) & 1));
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (rows b), column half w / 4
    uint64_t pw[7];
    pw[0] = 1 % m;
    for (int s = 1; s < 7; ++s) pw[s] = mm_red(pw[s - 1] << 8, m, mu);
    const int lq = warp & 3, half = warp >> 2;
    const int b = b0 + lq * 32 + lane;
    for (int cc = 0; cc < 2; ++cc) {
        const int col = half * 32 + cc * 16;
        uint64_t acc[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) acc[t] = 0;
#pragma unroll
        for (int s = 0; s < 7; ++s) {
            uint32_t v[16];
            const uint32_t ta = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(s * TC_N + col);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int t = 0; t < 16; ++t) acc[t] += (uint64_t)v[t] * pw[s];
        }
        if (b < n.B) {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int j = j0 + col + t;
                if (j >= wj) continue;
                const int jo = n.out_perm ? n.out_perm[uint64_t(r) * wj + j] : j;
                n.out[((uint64_t(k) * n.d + r) * n.out_bm + (n.out_bm > 1 ? b : 0)) * wj + jo] = mm_red(acc[t], m, mu);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// Byte-plane operands in global memory, pre-tiled in the canonical UMMA K-major layout so the
// GEMM streams them with 1-D bulk copies (TMA engine, no register traffic): one 32 KB chunk
// per (modulus k, row r, 128-row b tile, 64-i block) for x (4 planes x 128 x 64 B) and one
// 16 KB chunk per (k, r, 64-column j tile, 64-i block) for M (4 planes x 64 x 64 B).
__global__ void k_planes_x(const __grid_constant__ Node n, int qc, int K, int nbt, int nkb, unsigned char *out) {
    const int wi = n.w[qc];
    const uint64_t items = uint64_t(K) * n.d * nbt * TC_M * (nkb * 4);   // (kr, row, 16-i chunk)
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < items; e += uint64_t(gridDim.x) * blockDim.x) {
        const int row = (int)(e % TC_M);
        uint64_t t = e / TC_M;
        const int c16 = (int)(t % (nkb * 4));
        t /= (nkb * 4);
        const int bt = (int)(t % nbt);
        const int kr = (int)(t / nbt);
        const int k = kr / n.d, r = kr % n.d;
        const int b = bt * TC_M + row, ib = c16 * 16;
        uint32_t w[4][4];
        const uint64_t *x = (b < n.B) ? msg_row(n, qc, k, r, b, 0) : nullptr;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = ib + q * 4 + u;
                v[u] = (x && i < wi) ? (uint32_t)__ldg(reinterpret_cast<const unsigned long long *>(x) + i) : 0u;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
                w[a][q] = ((v[0] >> (8 * a)) & 0xFF) | (((v[1] >> (8 * a)) & 0xFF) << 8) | (((v[2] >> (8 * a)) & 0xFF) << 16) |
                          (((v[3] >> (8 * a)) & 0xFF) << 24);
        }
        const int kb = c16 >> 2, c = c16 & 3;
        unsigned char *chunk = out + ((uint64_t(kr) * nbt + bt) * nkb + kb) * (4 * TC_A_PLANE);
        const int off = c * (TC_M * 16) + (row >> 3) * 128 + (row & 7) * 16;
#pragma unroll
        for (int a = 0; a < 4; ++a)
            *reinterpret_cast<uint4 *>(chunk + a * TC_A_PLANE + off) = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
    }
}
__global__ void k_planes_m(const uint32_t *Rc, int Kd, int wi, int wj, int njt, int nkb, unsigned char *out) {
    const uint64_t items = uint64_t(Kd) * njt * TC_N * (nkb * 4);   // (kr, j, 16-i chunk); j fastest (coalesced reads)
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < items; e += uint64_t(gridDim.x) * blockDim.x) {
        const int jr = (int)(e % TC_N);
        uint64_t t = e / TC_N;
        const int jt = (int)(t % njt);
        t /= njt;
        const int c16 = (int)(t % (nkb * 4));
        const int kr = (int)(t / (nkb * 4));
        const int j = jt * TC_N + jr, ib = c16 * 16;
        const uint32_t *R = Rc + uint64_t(kr) * wi * wj;
        uint32_t w[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = ib + q * 4 + u;
                v[u] = (j < wj && i < wi) ? __ldg(R + uint64_t(i) * wj + j) : 0u;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
                w[a][q] = ((v[0] >> (8 * a)) & 0xFF) | (((v[1] >> (8 * a)) & 0xFF) << 8) | (((v[2] >> (8 * a)) & 0xFF) << 16) |
                          (((v[3] >> (8 * a)) & 0xFF) << 24);
        }
        // the 4 limb planes stacked along N (row a * 64 + j of one 256-row K-major operand,
        // 16-byte K chunks 4096 B apart): one N = 256 MMA per x limb covers all 4 M limbs
        const int kb = c16 >> 2, c = c16 & 3;
        unsigned char *chunk = out + ((uint64_t(kr) * njt + jt) * nkb + kb) * (4 * TC_B_PLANE);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int jj = a * TC_N + jr;
            *reinterpret_cast<uint4 *>(chunk + c * (4 * TC_N * 16) + (jj >> 3) * 128 + (jj & 7) * 16) =
                make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
        }
    }
}

// The tensor-core GEMM fed by bulk copies, persistent: one CTA per SM walks the (k r, b tile,
// j tile) tiles with a static stride.  Warp 4 (one lane) streams the pre-tiled x and M chunks
// of every 64-i block of every tile into a 4-stage ring (mbarrier full[s], expect_tx 48 KB),
// running ahead across tile boundaries; warp 5 (one lane) waits full[s], issues the 32 MMAs
// and commits them to empty[s], and after a tile's last block commits tmem_full; warps 0-3
// drain the 7 accumulators (tcgen05.ld, one TMEM lane quarter each), form the residues, store
// them (16-byte vector stores when the row is contiguous) and release TMEM (tmem_empty) for
// the next tile's MMAs.
constexpr int TC_ST2 = 4;
constexpr int TC_SMEM2 = TC_ST2 * TC_STAGE + 128;
__global__ void __launch_bounds__(192, 1) k_node_mat_gemm_bulk(const __grid_constant__ Node n, const __grid_constant__ Mods md,
                                                               int qc, const unsigned char *Xp, const unsigned char *Mp,
                                                               int nbt, int njt, int nkb, int kr_m0) {
    extern __shared__ __align__(1024) unsigned char tsm[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tsm);
    const uint32_t full0 = sbase + TC_ST2 * TC_STAGE, empty0 = full0 + 8 * TC_ST2;
    const uint32_t tfull = empty0 + 8 * TC_ST2, tempty = tfull + 8, slot = tempty + 8;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wj = n.w[1 - qc];
    const int ntiles = n.d * md.K * nbt * njt;
    if (tid == 0) {
        for (int s = 0; s < TC_ST2; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * s) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8 * s) : "memory");
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tfull) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(tempty) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(slot) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t tmem;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(slot) : "memory");

    if (warp == 4) {
        if (lane == 0) {   // producer
            uint32_t g = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int jt = t % njt, bt = (t / njt) % nbt, kr = t / (njt * nbt);
                const unsigned char *xa = Xp + (uint64_t(kr) * nbt + bt) * nkb * (4 * TC_A_PLANE);
                const unsigned char *mb = Mp + (uint64_t(kr_m0 + kr) * njt + jt) * nkb * (4 * TC_B_PLANE);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const uint32_t st = g % TC_ST2;
                    if (g >= TC_ST2) tc_mbar_wait(empty0 + 8 * st, ((g / TC_ST2) - 1) & 1);
                    const uint32_t fb = full0 + 8 * st, dst = sbase + st * TC_STAGE;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"((uint32_t)TC_STAGE) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                                 "l"(xa + uint64_t(kb) * (4 * TC_A_PLANE)), "r"((uint32_t)(4 * TC_A_PLANE)), "r"(fb) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + 4 * TC_A_PLANE),
                                 "l"(mb + uint64_t(kb) * (4 * TC_B_PLANE)), "r"((uint32_t)(4 * TC_B_PLANE)), "r"(fb) : "memory");
                }
            }
        }
        __syncwarp();
    } else if (warp == 5) {
        if (lane == 0) {   // MMA issuer
            // x limb a times all 4 M limbs in one N = 256 MMA: columns [64 a, 64 a + 256) of TMEM
            // are exactly D_a .. D_{a+3}, so every product lands on its shift s = a + c
            const uint32_t idesc = (2u << 4) | ((uint32_t)((4 * TC_N) >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
            const uint32_t idesc3 = (2u << 4) | ((uint32_t)((3 * TC_N) >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
            const uint32_t idesc1 = (2u << 4) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
            uint32_t g = 0, li = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++li) {
                tc_mbar_wait(tempty, li & 1);   // the epilogue has read the previous tile
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const uint32_t st = g % TC_ST2;
                    tc_mbar_wait(full0 + 8 * st, (g / TC_ST2) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a_s = sbase + st * TC_STAGE, b_s = a_s + 4 * TC_A_PLANE;
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int ks = 0; ks < TC_KB / 32; ++ks) {
                            const uint64_t ad = tc_sdesc(a_s + a * TC_A_PLANE + ks * 2 * (TC_M * 16), TC_M * 16, 128);
                            const uint32_t bs = b_s + ks * 2 * (4 * TC_N * 16);
                            const uint32_t dt = tmem + (uint32_t)(a * TC_N);
                            if (kb == 0 && ks == 0 && a > 0) {
                                // first touch of D_{a+3}: M limbs 0-2 accumulate into D_a..D_{a+2},
                                // limb 3 overwrites D_{a+3} (no zeroing pass needed)
                                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                                             "l"(ad), "l"(tc_sdesc(bs, 4 * TC_N * 16, 128)), "r"(idesc3), "r"(1u) : "memory");
                                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt + (uint32_t)(3 * TC_N)),
                                             "l"(ad), "l"(tc_sdesc(bs + (3 * TC_N / 8) * 128, 4 * TC_N * 16, 128)), "r"(idesc1), "r"(0u)
                                             : "memory");
                            } else {
                                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
                                             "l"(ad), "l"(tc_sdesc(bs, 4 * TC_N * 16, 128)), "r"(idesc),
                                             "r"((kb == 0 && ks == 0) ? 0u : 1u) : "memory");
                            }
                        }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty0 + 8 * st) : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tfull) : "memory");
            }
        }
        __syncwarp();
    } else {   // epilogue: warps 0-3, TMEM lanes 32 w .. 32 w + 31 = rows b
        // release TMEM to the issuer (initially, then after each tile's last read)
        auto release_acc = [&]() {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty) : "memory");
        };
        release_acc();
        uint32_t li = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++li) {
            const int jt = t % njt, bt = (t / njt) % nbt, kr = t / (njt * nbt);
            const int k = kr / n.d, r = kr % n.d;
            const uint64_t m = md.m[k], mu = md.mu[k];
            uint64_t pw[7];
            pw[0] = 1 % m;
            for (int s = 1; s < 7; ++s) pw[s] = mm_red(pw[s - 1] << 8, m, mu);
            const int b = bt * TC_M + warp * 32 + lane, j0 = jt * TC_N;
            tc_mbar_wait(tfull, li & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint64_t *orow = n.out + ((uint64_t(k) * n.d + r) * n.out_bm + (n.out_bm > 1 ? b : 0)) * wj;
            for (int col = 0; col < TC_N; col += 16) {
                uint64_t acc[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) acc[u] = 0;
                // the 7 loads of this column chunk in flight together, one wait; the empty asm
                // ties the registers to the wait so no use is scheduled before it
                uint32_t v[7][16];
#pragma unroll
                for (int s = 0; s < 7; ++s) {
                    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(s * TC_N + col);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                                 : "=r"(v[s][0]), "=r"(v[s][1]), "=r"(v[s][2]), "=r"(v[s][3]), "=r"(v[s][4]), "=r"(v[s][5]),
                                   "=r"(v[s][6]), "=r"(v[s][7]), "=r"(v[s][8]), "=r"(v[s][9]), "=r"(v[s][10]), "=r"(v[s][11]),
                                   "=r"(v[s][12]), "=r"(v[s][13]), "=r"(v[s][14]), "=r"(v[s][15])
                                 : "r"(ta));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int s = 0; s < 7; ++s) {
                    asm volatile("" : "+r"(v[s][0]), "+r"(v[s][1]), "+r"(v[s][2]), "+r"(v[s][3]), "+r"(v[s][4]), "+r"(v[s][5]),
                                      "+r"(v[s][6]), "+r"(v[s][7]), "+r"(v[s][8]), "+r"(v[s][9]), "+r"(v[s][10]), "+r"(v[s][11]),
                                      "+r"(v[s][12]), "+r"(v[s][13]), "+r"(v[s][14]), "+r"(v[s][15]));
#pragma unroll
                    for (int u = 0; u < 16; ++u) acc[u] += (uint64_t)v[s][u] * pw[s];
                }
                if (col + 16 == TC_N) release_acc();   // every accumulator column read
                if (b < n.B) {
                    const int jb = j0 + col;
#pragma unroll
                    for (int u = 0; u < 16; ++u) acc[u] = mm_red(acc[u], m, mu);
                    if (!n.out_perm && jb + 16 <= wj) {
#pragma unroll
                        for (int u = 0; u < 16; u += 2)
                            *reinterpret_cast<ulonglong2 *>(orow + jb + u) = make_ulonglong2(acc[u], acc[u + 1]);
                    } else {
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int j = jb + u;
                            if (j >= wj) continue;
                            orow[n.out_perm ? n.out_perm[uint64_t(r) * wj + j] : j] = acc[u];
                        }
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// Matrix node with one child leg and one parent leg, one conditioned bucket (chains, PAPER.md
// :222-225): out[k][r][o] = sum_i x[k][r][i] * M(i, o) mod m_k for every modulus k in one pass
// over the matrix (each element is reduced once per modulus; the int64 matrix is read once per
// group of 8 moduli).  Block = 32 outputs (lanes) x 8 slices of the child index (warps); the
// slices' partial sums are combined in shared memory.  Residues < 2^26: products < 2^52, so up
// to 4096 of them accumulate exactly in 64 bits between reductions.
constexpr int MV_OUT = 32, MV_SL = 8, MV_G = 8;
__global__ void __launch_bounds__(256) k_node_matvec(const __grid_constant__ Node n, const __grid_constant__ Mods md, int qc) {
    __shared__ uint64_t part[MV_SL][MV_G][MV_OUT];
    const int r = blockIdx.x;
    const int qp = 1 - qc;
    const int wi = n.w[qc], wo = n.w[qp];
    const int lane = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int o = blockIdx.y * MV_OUT + lane;
    const int64_t *T = n.data[0] + uint64_t(r) * n.w[0] * n.w[1];
    const int chunk = (wi + MV_SL - 1) / MV_SL;
    const int i0 = sl * chunk, i1 = min(wi, i0 + chunk);
    for (int g0 = 0; g0 < md.K; g0 += MV_G) {
        const int ng = min(MV_G, md.K - g0);
        uint64_t acc[MV_G];
#pragma unroll
        for (int g = 0; g < MV_G; ++g) acc[g] = 0;
        if (o < wo) {
            for (int i = i0; i < i1; ++i) {
                const int64_t v = qc == 0 ? T[uint64_t(i) * wo + o] : T[uint64_t(o) * wi + i];
                const uint64_t av = uabs(v);
#pragma unroll
                for (int g = 0; g < MV_G; ++g) {
                    if (g >= ng) break;
                    const int k = g0 + g;
                    uint64_t rv = mm_red(av, md.m[k], md.mu[k]);
                    if (v < 0 && rv) rv = md.m[k] - rv;
                    acc[g] += rv * __ldg(reinterpret_cast<const unsigned long long *>(msg_row(n, qc, k, r, 0, 0)) + i);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < MV_G; ++g) part[sl][g][lane] = g < ng ? mm_red(acc[g], md.m[g0 + g], md.mu[g0 + g]) : 0;
        __syncthreads();
        // warp sl finishes modulus g = sl of this group for the block's 32 outputs
        if (sl < ng && o < wo) {
            const int k = g0 + sl;
            uint64_t t = 0;
            for (int s2 = 0; s2 < MV_SL; ++s2) t = mm_add(t, part[s2][sl][lane], md.m[k]);
            const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
            n.out[(uint64_t(k) * n.d + r) * n.out_bm * wo + oo] = t;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- exact int128 engine
// When the rigorous bound prod_t ||T_t||_1 is <= 2^125, every message,
// prefix sum and partial sum of a sub-plan without matrices is a signed sum of a subset of
// the expansion's terms, so it fits int128: the contraction runs once in exact int128
// arithmetic instead of once per CRT modulus.  Same node model and layouts as the modular
// kernels with K = 1 and 16-byte entries.
typedef __int128 i128;

__device__ __forceinline__ i128 shfl_xor_i128(i128 v, int o) {
    const uint64_t lo = __shfl_xor_sync(0xffffffffu, (uint64_t)v, o);
    const uint64_t hi = __shfl_xor_sync(0xffffffffu, (uint64_t)((unsigned __int128)v >> 64), o);
    return (i128)(((unsigned __int128)hi << 64) | lo);
}
__device__ __forceinline__ i128 shfl_up_i128(i128 v, int o) {
    const uint64_t lo = __shfl_up_sync(0xffffffffu, (uint64_t)v, o);
    const uint64_t hi = __shfl_up_sync(0xffffffffu, (uint64_t)((unsigned __int128)v >> 64), o);
    return (i128)(((unsigned __int128)hi << 64) | lo);
}
__device__ __forceinline__ i128 block_sum_i128(i128 v, i128 *red) {
    for (int o = 16; o > 0; o >>= 1) v += shfl_xor_i128(v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    i128 t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    return t;
}
// exact messages: int128, or int64 when the producing node's bound is <= 2^61 (narrow merged
// nodes; half the bytes written and read).  Read-only within a kernel (ld.global.nc).
struct MsgX {
    const void *p;
    bool w64;
    __device__ __forceinline__ i128 operator[](uint64_t i) const {
        if (w64) return (i128)__ldg(reinterpret_cast<const long long *>(p) + i);
        const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(p) + i);
        return (i128)(((unsigned __int128)(unsigned long long)v.y << 64) | (unsigned long long)v.x);
    }
    __device__ __forceinline__ explicit operator bool() const { return p != nullptr; }
};
__device__ __forceinline__ MsgX msg_row_x(const Node &n, int q, int r, int bb) {
    const int bm = n.bm[q];
    const uint64_t off = (uint64_t(r) * bm + (bm > 1 ? bb : 0)) * (uint64_t)n.w[q];
    const bool w64 = (n.m64 >> q) & 1;
    return MsgX{w64 ? (const void *)(reinterpret_cast<const int64_t *>(n.msg[q]) + off)
                    : (const void *)(reinterpret_cast<const i128 *>(n.msg[q]) + off), w64};
}
__device__ __forceinline__ void store_msg_x(const Node &n, uint64_t idx, i128 v) {
    if (n.out64) reinterpret_cast<int64_t *>(n.out)[idx] = (int64_t)v;
    else reinterpret_cast<i128 *>(n.out)[idx] = v;
}

// VEC / MAT node or merged leaf, exact.  blockIdx.x = r*B + bb, blockIdx.y = tile.
__global__ void k_node_dense_x(const __grid_constant__ Node n) {
    __shared__ i128 red[32];
    const int B = n.B;
    const int bb = blockIdx.x % B;
    const int r = blockIdx.x / B;
    const int64_t b = n.b0 + bb;
    int qp = -1, qf = -1, qc0 = -1, qc1 = -1;
    for (int q = 0; q < n.nl; ++q) {
        if (n.role[q] == RPARENT) qp = q;
        else if (n.role[q] == RFIXED) qf = q;
        else if (qc0 < 0) qc0 = q;
        else qc1 = q;
    }
    const int qo = qp >= 0 ? qp : qc0;
    const int qi = qp >= 0 ? qc0 : qc1;
    const int wo = qo >= 0 ? n.w[qo] : 1;
    const int wi = qi >= 0 ? n.w[qi] : 1;
    const MsgX xo = (qo >= 0 && n.role[qo] == RCHILD) ? msg_row_x(n, qo, r, bb) : MsgX{nullptr, false};
    const MsgX xi = (qi >= 0) ? msg_row_x(n, qi, r, bb) : MsgX{nullptr, false};
    i128 acc = 0;
    const int per_tile = (wo + n.tiles - 1) / n.tiles;
    const int o_begin = blockIdx.y * per_tile, o_end = min(wo, o_begin + per_tile);
    for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
        i128 s = 0;
        for (int i = 0; i < wi; ++i) {
            int64_t idx[3] = {0, 0, 0};
            if (qo >= 0) idx[qo] = o;
            if (qi >= 0) idx[qi] = i;
            if (qf >= 0) idx[qf] = b;
            i128 term = (i128)tensor_val(n, r, idx);
            if (xi) term *= xi[i];
            s += term;
        }
        if (qp >= 0) {
            const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
            store_msg_x(n, (uint64_t(r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo, s);
        } else {
            if (xo) s *= xo[o];
            acc += s;
        }
    }
    if (qp < 0) {
        const i128 t = block_sum_i128(acc, red);
        if (threadIdx.x == 0) reinterpret_cast<i128 *>(n.out)[(uint64_t(r) * B + bb) * n.tiles + blockIdx.y] = t;
    }
}

// per (row, outer index) threshold positions of a merged node whose contracted leg's
// thresholds depend on the outer index only (no fixed leg, no inner leg): computed once and
// shared by every conditioned bucket and every modulus.  pos = nless | nle << 16.
__global__ void k_merged_pos(const __grid_constant__ Node n, int qo, uint32_t *pos) {
    const int r = blockIdx.y;
    const int wo = n.w[qo], wq = n.w[n.qc];
    const uint64_t *S = n.sabs + uint64_t(r) * wq;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < wo; o += gridDim.x * blockDim.x) {
        bool hasL, hasR;
        int64_t L, R;
        merged_LR(n, r, n.qc, -1, qo, -1, 0, o, 0, hasL, L, hasR, R);
        const int nless = hasL ? count_lt(S, wq, uabs(L)) : 0;
        const int nle = hasR ? count_le(S, wq, uabs(R)) : 0;
        pos[uint64_t(r) * wo + o] = (uint32_t)nless | ((uint32_t)nle << 16);
    }
}

__device__ __forceinline__ i128 shfl_up_w(i128 v, int o) { return shfl_up_i128(v, o); }
__device__ __forceinline__ int64_t shfl_up_w(int64_t v, int o) { return __shfl_up_sync(0xffffffffu, (long long)v, o); }
__device__ __forceinline__ i128 shfl_xor_w(i128 v, int o) { return shfl_xor_i128(v, o); }
__device__ __forceinline__ int64_t shfl_xor_w(int64_t v, int o) { return __shfl_xor_sync(0xffffffffu, (long long)v, o); }
__device__ __forceinline__ int64_t shfl_idx_w(int64_t v, int l) { return __shfl_sync(0xffffffffu, (long long)v, l); }
__device__ __forceinline__ i128 shfl_idx_w(i128 v, int l) {
    const uint64_t lo = __shfl_sync(0xffffffffu, (unsigned long long)(uint64_t)v, l);
    const uint64_t hi = __shfl_sync(0xffffffffu, (unsigned long long)(uint64_t)((unsigned __int128)v >> 64), l);
    return (i128)(((unsigned __int128)hi << 64) | lo);
}
template <typename W>
__device__ __forceinline__ W block_sum_w(W v, W *red) {
    for (int o = 16; o > 0; o >>= 1) v += shfl_xor_w(v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    W t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    return t;
}

// prefix arrays of the exact merged kernel are padded by one slot every 8 entries (index s
// lives at PXI(s)), so each thread's contiguous chunk is read without bank conflicts
__device__ __forceinline__ int PXI(int s) { return s + (s >> 3); }

template <typename W>
__device__ __forceinline__ W o9_value_x(const W *P1, const W *P2, int wq, bool hasL, int64_t L, bool hasR,
                                        int64_t R, int nless, int nle) {
    W V;
    if (hasL) {
        const int64_t win = (hasR && !(uabs(L) <= uabs(R))) ? R : L;
        V = (W)win * (P1[PXI(wq)] - P1[PXI(nless)]);
        int endB = nless;
        if (hasR && nle < endB) {
            V += (W)R * (P1[PXI(endB)] - P1[PXI(nle)]);
            endB = nle;
        }
        V += P2[PXI(endB)];
    } else {
        V = (W)R * (P1[PXI(wq)] - P1[PXI(nle)]) + P2[PXI(nle)];
    }
    return V;
}

// merged node, exact: prefix sums P1 (x) and P2 (x*c) over the |c|-sorted contracted leg in
// shared memory (block scan), then O(1) per output.  pos_pre: precomputed
// thresholds (k_merged_pos) or null (binary searches over the sorted |c| in global memory).
constexpr int MX_T = 512;
// W = i128, or int64_t when the node's message-passing bound (F_t x its children's message
// bounds) is below 2^62: half the shared memory (two CTAs per SM) and 64-bit
// arithmetic; messages in memory stay int128.
template <typename W>
__global__ void __launch_bounds__(MX_T) k_node_merged_x(const __grid_constant__ Node n, const uint32_t *pos_pre) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ W red[32];
    __shared__ W tot1[32], tot2[32];
    const int B = n.B;
    const int bb = blockIdx.x % B;
    const int r = blockIdx.x / B;
    const int64_t b = n.b0 + bb;
    const int qc = n.qc;
    const int wq = n.w[qc];
    W *P1 = reinterpret_cast<W *>(sm);
    W *P2 = P1 + (PXI(wq) + 1);
    const int64_t *cs = n.csorted + uint64_t(r) * wq;
    const uint64_t *S = n.sabs + uint64_t(r) * wq;
    int qp = -1, qf = -1, oc[2] = {-1, -1}, noc = 0;
    for (int q = 0; q < n.nl; ++q) {
        if (q == qc) continue;
        if (n.role[q] == RPARENT) qp = q;
        else if (n.role[q] == RFIXED) qf = q;
        else oc[noc++] = q;
    }
    const int qo = qp >= 0 ? qp : oc[0];
    const int qi = qp >= 0 ? oc[0] : oc[1];
    const int wo = qo >= 0 ? n.w[qo] : 1;
    const int wi = qi >= 0 ? n.w[qi] : 1;
    const int per_tile = (wo + n.tiles - 1) / n.tiles;
    const int o_begin = blockIdx.y * per_tile, o_end = min(wo, o_begin + per_tile);
    // --- prefix sums over the |c|-sorted order: the terms x and x*c are staged in P1 / P2
    //     with coalesced loads (the message is read once); thread t then scans its contiguous
    //     chunk in registers, one warp shuffle scan combines the thread totals, thread 0 scans
    //     the warp totals, and each thread writes its chunk's exclusive prefixes back
    const MsgX x = msg_row_x(n, qc, r, bb);   // delivered in the |c|-sorted order
    for (int s = threadIdx.x; s < wq; s += MX_T) {
        const W xv = (W)x[s];
        P1[PXI(s)] = xv;
        P2[PXI(s)] = xv * (W)cs[s];
    }
    __syncthreads();
    {
        constexpr int NW = MX_T / 32;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const int ch = (wq + MX_T - 1) / MX_T;
        const int s0 = min(wq, (int)threadIdx.x * ch), s1 = min(wq, s0 + ch);
        W t1 = 0, t2 = 0;
        for (int s = s0; s < s1; ++s) { t1 += P1[PXI(s)]; t2 += P2[PXI(s)]; }
        W i1 = t1, i2 = t2;
        for (int o = 1; o < 32; o <<= 1) {
            const W u1 = shfl_up_w(i1, o), u2 = shfl_up_w(i2, o);
            if (lane >= o) { i1 += u1; i2 += u2; }
        }
        if (lane == 31) { tot1[wid] = i1; tot2[wid] = i2; }
        __syncthreads();
        if (threadIdx.x == 0) {
            W e1 = 0, e2 = 0;
            for (int w = 0; w < NW; ++w) {
                const W a1 = tot1[w], a2 = tot2[w];
                tot1[w] = e1;
                tot2[w] = e2;
                e1 += a1;
                e2 += a2;
            }
            P1[PXI(wq)] = e1;
            P2[PXI(wq)] = e2;
        }
        __syncthreads();
        W c1 = tot1[wid] + i1 - t1, c2 = tot2[wid] + i2 - t2;   // exclusive prefix at s0
        for (int s = s0; s < s1; ++s) {
            const W v1 = P1[PXI(s)], v2 = P2[PXI(s)];
            P1[PXI(s)] = c1;
            P2[PXI(s)] = c2;
            c1 += v1;
            c2 += v2;
        }
    }
    __syncthreads();
    // --- outputs
    const MsgX xo = (qo >= 0 && n.role[qo] == RCHILD) ? msg_row_x(n, qo, r, bb) : MsgX{nullptr, false};
    const MsgX xi2 = qi >= 0 ? msg_row_x(n, qi, r, bb) : MsgX{nullptr, false};
    W acc = 0;
    // no inner leg and rank tables present (the common case): the fixed leg's value and rank
    // are loop invariants, only the outer leg's constituent varies per output
    const bool ranked = n.rank[0] || n.rank[1] || n.rank[2];
    if (qi < 0 && ranked) {
        const bool hasF = qf >= 0, fL = hasF && qf < qc, oL = qo >= 0 && qo < qc;
        const int64_t vf = hasF ? n.data[qf][uint64_t(r) * n.w[qf] + b] : 0;
        const uint32_t rf = hasF ? n.rank[qf][uint64_t(r) * n.w[qf] + b] : 0u;
        const int64_t *dO = qo >= 0 ? n.data[qo] + uint64_t(r) * wo : nullptr;
        const uint32_t *rO = qo >= 0 ? n.rank[qo] + uint64_t(r) * wo : nullptr;
        const bool f_first = hasF && qo >= 0 && qf < qo;   // fold order when both sit on one side
        // read-only loads (ld.global.nc) so the loads of later outputs are not held behind this
        // thread's message stores; unrolled for several outputs in flight
#pragma unroll 4
        for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
            int64_t vo = 0;
            uint32_t ro = 0;
            if (qo >= 0) { vo = __ldg(reinterpret_cast<const long long *>(dO) + o); ro = __ldg(rO + o); }
            bool hasL = false, hasR = false;
            int64_t L = 0, R = 0;
            uint32_t rL = 0, rR = 0;
            if (hasF && qo >= 0 && fL == oL) {   // both on one side: left fold in leg order
                const int64_t a = f_first ? vf : vo, c = f_first ? vo : vf;
                const uint32_t ra = f_first ? rf : ro, rc = f_first ? ro : rf;
                const bool keep = uabs(a) <= uabs(c);
                if (fL) { hasL = true; L = keep ? a : c; rL = keep ? ra : rc; }
                else { hasR = true; R = keep ? a : c; rR = keep ? ra : rc; }
            } else {
                if (hasF) { if (fL) { hasL = true; L = vf; rL = rf; } else { hasR = true; R = vf; rR = rf; } }
                if (qo >= 0) { if (oL) { hasL = true; L = vo; rL = ro; } else { hasR = true; R = vo; rR = ro; } }
            }
            const int nless = hasL ? (int)(rL & 0xffffu) : 0, nle = hasR ? (int)(rR >> 16) : 0;
            W sacc = o9_value_x<W>(P1, P2, wq, hasL, L, hasR, R, nless, nle);
            if (qp >= 0) {
                const int oo = n.out_perm ? __ldg(n.out_perm + uint64_t(r) * wo + o) : o;
                store_msg_x(n, (uint64_t(r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo, (i128)sacc);
            } else {
                if (xo) sacc *= (W)xo[o];
                acc += sacc;
            }
        }
    } else
    for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
        W sacc = 0;
        for (int i = 0; i < wi; ++i) {
            bool hasL, hasR;
            int64_t L, R;
            int nless, nle;
            merged_thr(n, r, qc, qf, qo, qi, b, o, i, S, wq, hasL, L, hasR, R, nless, nle);
            W V = o9_value_x<W>(P1, P2, wq, hasL, L, hasR, R, nless, nle);
            if (xi2) V *= (W)xi2[i];
            sacc += V;
        }
        if (qp >= 0) {
            const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
            store_msg_x(n, (uint64_t(r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo, (i128)sacc);
        } else {
            if (xo) sacc *= (W)xo[o];
            acc += sacc;
        }
    }
    if (qp < 0) {
        const W t = block_sum_w(acc, red);
        if (threadIdx.x == 0) reinterpret_cast<i128 *>(n.out)[(uint64_t(r) * B + bb) * n.tiles + blockIdx.y] = (i128)t;
    }
}

// merged node, modular (CRT engine): the same structure as k_node_merged_x — thresholds once
// per block (or precomputed per node), then per modulus a block scan (warp 0 scans the
// per-thread totals with shuffles) and O(1) work per output.
__device__ __forceinline__ uint64_t shfl_up_mod_scan(uint64_t v, int lane, uint64_t m) {
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = mm_add(v, u, m);
    }
    return v;
}
__global__ void __launch_bounds__(MX_T) k_node_merged_m(const __grid_constant__ Node n, const __grid_constant__ Mods md,
                                                        const uint32_t *pos_pre) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ uint64_t red[32];
    __shared__ uint64_t tot1[MX_T], tot2[MX_T];
    const int B = n.B;
    const int bb = blockIdx.x % B;
    const int r = blockIdx.x / B;
    const int64_t b = n.b0 + bb;
    const int qc = n.qc;
    const int wq = n.w[qc];
    uint64_t *P1 = reinterpret_cast<uint64_t *>(sm);
    uint64_t *P2 = P1 + (wq + 1);
    uint32_t *pos = reinterpret_cast<uint32_t *>(P2 + (wq + 1));   // per outer index of this tile (no inner leg)
    const int64_t *cs = n.csorted + uint64_t(r) * wq;
    const uint64_t *S = n.sabs + uint64_t(r) * wq;
    int qp = -1, qf = -1, oc[2] = {-1, -1}, noc = 0;
    for (int q = 0; q < n.nl; ++q) {
        if (q == qc) continue;
        if (n.role[q] == RPARENT) qp = q;
        else if (n.role[q] == RFIXED) qf = q;
        else oc[noc++] = q;
    }
    const int qo = qp >= 0 ? qp : oc[0];
    const int qi = qp >= 0 ? oc[0] : oc[1];
    const int wo = qo >= 0 ? n.w[qo] : 1;
    const int wi = qi >= 0 ? n.w[qi] : 1;
    const int per_tile = (wo + n.tiles - 1) / n.tiles;
    const int o_begin = blockIdx.y * per_tile, o_end = min(wo, o_begin + per_tile);
    const bool cache_pos = qi < 0;
    if (cache_pos) {
        for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
            if (pos_pre) { pos[o - o_begin] = pos_pre[uint64_t(r) * wo + o]; continue; }
            bool hasL, hasR;
            int64_t L, R;
            int nless, nle;
            merged_thr(n, r, qc, qf, qo, qi, b, o, 0, S, wq, hasL, L, hasR, R, nless, nle);
            pos[o - o_begin] = (uint32_t)nless | ((uint32_t)nle << 16);
        }
    }
    const int chunk = (wq + MX_T - 1) / MX_T;
    const int s0 = threadIdx.x * chunk, s1 = min(wq, s0 + chunk);
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < md.K; ++k) {
        const uint64_t m = md.m[k], mu = md.mu[k];
        const uint64_t *x = msg_row(n, qc, k, r, bb, 0);   // |c|-sorted order
        uint64_t l1 = 0, l2 = 0;
        for (int s = s0; s < s1; ++s) {
            const uint64_t xv = x[s];
            l1 += xv;                                   // < chunk * 2^26: reduced once below
            l2 = mm_add(l2, mm_mul(xv, mm_i64(cs[s], m, mu), m, mu), m);
        }
        __syncthreads();   // previous modulus finished with P1/P2/tot
        tot1[threadIdx.x] = mm_red(l1, m, mu);
        tot2[threadIdx.x] = l2;
        __syncthreads();
        if (threadIdx.x < 32) {
            constexpr int per = MX_T / 32;
            uint64_t a1 = 0, a2 = 0;
            for (int t = 0; t < per; ++t) { a1 = mm_add(a1, tot1[lane * per + t], m); a2 = mm_add(a2, tot2[lane * per + t], m); }
            const uint64_t i1 = shfl_up_mod_scan(a1, lane, m), i2 = shfl_up_mod_scan(a2, lane, m);
            uint64_t e1 = mm_sub(i1, a1, m), e2 = mm_sub(i2, a2, m);
            for (int t = 0; t < per; ++t) {
                const uint64_t v1 = tot1[lane * per + t], v2 = tot2[lane * per + t];
                tot1[lane * per + t] = e1;
                tot2[lane * per + t] = e2;
                e1 = mm_add(e1, v1, m);
                e2 = mm_add(e2, v2, m);
            }
            if (lane == 31) { P1[wq] = i1; P2[wq] = i2; }
        }
        __syncthreads();
        {
            uint64_t c1 = tot1[threadIdx.x], c2 = tot2[threadIdx.x];
            for (int s = s0; s < s1; ++s) {
                P1[s] = c1;
                P2[s] = c2;
                const uint64_t xv = x[s];
                c1 = mm_add(c1, xv, m);
                c2 = mm_add(c2, mm_mul(xv, mm_i64(cs[s], m, mu), m, mu), m);
            }
        }
        __syncthreads();
        const uint64_t *xo = (qo >= 0 && n.role[qo] == RCHILD) ? msg_row(n, qo, k, r, bb, 0) : nullptr;
        const uint64_t *xi2 = qi >= 0 ? msg_row(n, qi, k, r, bb, 0) : nullptr;
        uint64_t acc = 0;
        for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
            uint64_t sacc = 0;
            for (int i = 0; i < wi; ++i) {
                bool hasL, hasR;
                int64_t L, R;
                int nless, nle;
                if (cache_pos) {
                    merged_LR(n, r, qc, qf, qo, qi, b, o, i, hasL, L, hasR, R);
                    const uint32_t pv = pos[o - o_begin];
                    nless = (int)(pv & 0xffffu);
                    nle = (int)(pv >> 16);
                } else {
                    merged_thr(n, r, qc, qf, qo, qi, b, o, i, S, wq, hasL, L, hasR, R, nless, nle);
                }
                uint64_t V = o9_value(P1, P2, wq, hasL, L, hasR, R, nless, nle, m, mu);
                if (xi2) V = mm_mul(V, xi2[i], m, mu);
                sacc = mm_add(sacc, V, m);
            }
            if (qp >= 0) {
                const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
                n.out[((uint64_t(k) * n.d + r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo] = sacc;
            } else {
                if (xo) sacc = mm_mul(sacc, xo[o], m, mu);
                acc = mm_add(acc, sacc, m);
            }
        }
        if (qp < 0) {
            const uint64_t t = block_sum_mod(acc, m, red);
            if (threadIdx.x == 0) n.out[((uint64_t(k) * n.d + r) * B + bb) * n.tiles + blockIdx.y] = t;
        }
    }
}

// ---------------------------------------------------------------- absolute-value bound pass
// |E_r| <= A_r = the same contraction with every tensor entry replaced by its absolute value
// (a merged view's entry by min_q |v_q|).  All quantities are non-negative, so the fp64 pass
// uses sums and products only (prefix sums of x*c and suffix sums of x — no differences):
// V(o) = sum_s x_s min(t_o, c_s) = P2[n_t] + t_o * SUF1[n_t], t_o = min |other legs|,
// n_t = #{c_s < t_o}.  The relative rounding error of such a computation is below 2^-26 here
// (< 2^27 sequential additions on any path), so A_r (1 + 2^-16) bounds |E_r| rigorously; it is
// far tighter than prod_t ||T_t||_1 (one index per edge instead of one per table leg), which
// lets most merged sub-plans run on the exact int128 engine.
__device__ __forceinline__ double block_sum_f64(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    return t;
}
__device__ __forceinline__ const double *msg_row_a(const Node &n, int q, int r, int bb) {
    const int bm = n.bm[q];
    return reinterpret_cast<const double *>(n.msg[q]) + (uint64_t(r) * bm + (bm > 1 ? bb : 0)) * (uint64_t)n.w[q];
}
__device__ __forceinline__ double tensor_abs(const Node &n, int r, const int64_t *idx) {
    if (n.kind == KV) return (double)uabs(n.data[0][uint64_t(r) * n.w[0] + idx[0]]);
    if (n.kind == KM) return (double)uabs(n.data[0][(uint64_t(r) * n.w[0] + idx[0]) * n.w[1] + idx[1]]);
    uint64_t m = uabs(n.data[0][uint64_t(r) * n.w[0] + idx[0]]);
    for (int q = 1; q < n.nl; ++q) m = min(m, uabs(n.data[q][uint64_t(r) * n.w[q] + idx[q]]));
    return (double)m;
}

__global__ void k_node_dense_abs(const __grid_constant__ Node n) {
    __shared__ double red[32];
    const int B = n.B;
    const int bb = blockIdx.x % B;
    const int r = blockIdx.x / B;
    const int64_t b = n.b0 + bb;
    int qp = -1, qf = -1, qc0 = -1, qc1 = -1;
    for (int q = 0; q < n.nl; ++q) {
        if (n.role[q] == RPARENT) qp = q;
        else if (n.role[q] == RFIXED) qf = q;
        else if (qc0 < 0) qc0 = q;
        else qc1 = q;
    }
    const int qo = qp >= 0 ? qp : qc0;
    const int qi = qp >= 0 ? qc0 : qc1;
    const int wo = qo >= 0 ? n.w[qo] : 1;
    const int wi = qi >= 0 ? n.w[qi] : 1;
    const double *xo = (qo >= 0 && n.role[qo] == RCHILD) ? msg_row_a(n, qo, r, bb) : nullptr;
    const double *xi = (qi >= 0) ? msg_row_a(n, qi, r, bb) : nullptr;
    double acc = 0;
    const int per_tile = (wo + n.tiles - 1) / n.tiles;
    const int o_begin = blockIdx.y * per_tile, o_end = min(wo, o_begin + per_tile);
    for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
        double s = 0;
        for (int i = 0; i < wi; ++i) {
            int64_t idx[3] = {0, 0, 0};
            if (qo >= 0) idx[qo] = o;
            if (qi >= 0) idx[qi] = i;
            if (qf >= 0) idx[qf] = b;
            double term = tensor_abs(n, r, idx);
            if (xi) term *= xi[i];
            s += term;
        }
        if (qp >= 0) {
            const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
            reinterpret_cast<double *>(n.out)[(uint64_t(r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo] = s;
        } else {
            if (xo) s *= xo[o];
            acc += s;
        }
    }
    if (qp < 0) {
        const double t = block_sum_f64(acc, red);
        if (threadIdx.x == 0) reinterpret_cast<double *>(n.out)[(uint64_t(r) * B + bb) * n.tiles + blockIdx.y] = t;
    }
}

__global__ void __launch_bounds__(MX_T) k_node_merged_abs(const __grid_constant__ Node n) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[32];
    __shared__ double tot1[MX_T], tot2[MX_T];
    const int B = n.B;
    const int bb = blockIdx.x % B;
    const int r = blockIdx.x / B;
    const int64_t b = n.b0 + bb;
    const int qc = n.qc;
    const int wq = n.w[qc];
    double *P2 = reinterpret_cast<double *>(sm);     // prefix sums of x*|c|   [wq + 1]
    double *S1 = P2 + (wq + 1);                      // suffix sums of x       [wq + 1]
    const int64_t *cs = n.csorted + uint64_t(r) * wq;
    const uint64_t *S = n.sabs + uint64_t(r) * wq;
    int qp = -1, qf = -1, oc[2] = {-1, -1}, noc = 0;
    for (int q = 0; q < n.nl; ++q) {
        if (q == qc) continue;
        if (n.role[q] == RPARENT) qp = q;
        else if (n.role[q] == RFIXED) qf = q;
        else oc[noc++] = q;
    }
    const int qo = qp >= 0 ? qp : oc[0];
    const int qi = qp >= 0 ? oc[0] : oc[1];
    const int wo = qo >= 0 ? n.w[qo] : 1;
    const int wi = qi >= 0 ? n.w[qi] : 1;
    const int per_tile = (wo + n.tiles - 1) / n.tiles;
    const int o_begin = blockIdx.y * per_tile, o_end = min(wo, o_begin + per_tile);
    const double *x = msg_row_a(n, qc, r, bb);
    const int chunk = (wq + MX_T - 1) / MX_T;
    const int s0 = threadIdx.x * chunk, s1 = min(wq, s0 + chunk);
    double l1 = 0, l2 = 0;
    for (int s = s0; s < s1; ++s) { l1 += x[s]; l2 += x[s] * (double)uabs(cs[s]); }
    tot1[threadIdx.x] = l1;
    tot2[threadIdx.x] = l2;
    __syncthreads();
    if (threadIdx.x == 0) {   // exclusive prefix (tot2) and suffix-after (tot1) of the thread totals
        double c2 = 0;
        for (int t = 0; t < MX_T; ++t) { const double v = tot2[t]; tot2[t] = c2; c2 += v; }
        P2[wq] = c2;
        double c1 = 0;
        for (int t = MX_T - 1; t >= 0; --t) { const double v = tot1[t]; tot1[t] = c1; c1 += v; }
        S1[wq] = 0;
    }
    __syncthreads();
    {
        double c2 = tot2[threadIdx.x];
        for (int s = s0; s < s1; ++s) { P2[s] = c2; c2 += x[s] * (double)uabs(cs[s]); }
        double c1 = tot1[threadIdx.x];
        for (int s = s1 - 1; s >= s0; --s) { c1 += x[s]; S1[s] = c1; }
    }
    __syncthreads();
    const double *xo = (qo >= 0 && n.role[qo] == RCHILD) ? msg_row_a(n, qo, r, bb) : nullptr;
    const double *xi2 = qi >= 0 ? msg_row_a(n, qi, r, bb) : nullptr;
    double acc = 0;
    for (int o = o_begin + threadIdx.x; o < o_end; o += blockDim.x) {
        double sacc = 0;
        for (int i = 0; i < wi; ++i) {
            uint64_t t = ~0ULL;   // min |value| over the other legs
            for (int q = 0; q < n.nl; ++q) {
                if (q == qc) continue;
                const int64_t ix = (q == qf) ? b : (q == qo ? o : i);
                t = min(t, uabs(n.data[q][uint64_t(r) * n.w[q] + ix]));
            }
            const int nt = count_lt(S, wq, t);
            double V = P2[nt] + (double)t * S1[nt];
            if (xi2) V *= xi2[i];
            sacc += V;
        }
        if (qp >= 0) {
            const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
            reinterpret_cast<double *>(n.out)[(uint64_t(r) * n.out_bm + (n.out_bm > 1 ? bb : 0)) * wo + oo] = sacc;
        } else {
            if (xo) sacc *= xo[o];
            acc += sacc;
        }
    }
    if (qp < 0) {
        const double t = block_sum_f64(acc, red);
        if (threadIdx.x == 0) reinterpret_cast<double *>(n.out)[(uint64_t(r) * B + bb) * n.tiles + blockIdx.y] = t;
    }
}

__global__ void k_root_reduce_abs(const double *part, double *acc, int slots) {
    __shared__ double red[32];
    double s = 0;
    for (int i = threadIdx.x; i < slots; i += blockDim.x) s += part[uint64_t(blockIdx.x) * slots + i];
    const double t = block_sum_f64(s, red);
    if (threadIdx.x == 0) acc[blockIdx.x] += t;
}

// acc[r] += sum over slots of part[r][slot], exact
__global__ void k_root_reduce_x(const i128 *part, i128 *acc, int slots) {
    __shared__ i128 red[32];
    i128 s = 0;
    for (int i = threadIdx.x; i < slots; i += blockDim.x) s += part[uint64_t(blockIdx.x) * slots + i];
    const i128 t = block_sum_i128(s, red);
    if (threadIdx.x == 0) acc[blockIdx.x] += t;
}

// Residues of a matrix node, child-leg major: Rc[k][r][i][o] = M(i, o) mod m_k (i = child-leg
// index, o = parent-leg index), computed once per (matrix, orientation) per estimate batch and
// shared by every chain sub-plan through that matrix.
__global__ void k_mat_residues(const int64_t *T, int d, int w0, int w1, int qc, const __grid_constant__ Mods md,
                               uint32_t *Rc) {
    // 32 x 32 tiles of row r (blockIdx.z) of the matrix, staged through shared memory so the
    // int64 reads and the K uint32 writes per element are both coalesced in either
    // orientation (Rc[k][r][i][o], i = the contracted leg); widths are powers of two
    __shared__ int64_t tile[32][33];
    const int wi = qc == 0 ? w0 : w1, wo = qc == 0 ? w1 : w0;
    const uint64_t cells = uint64_t(w0) * w1;
    const int r = blockIdx.z;
    const int64_t *Tr = T + uint64_t(r) * cells;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: 32 x 8
    const int ntx = (wo + 31) / 32;
    for (int tb = blockIdx.x; tb < ntx * ((wi + 31) / 32); tb += gridDim.x) {
        const int i0 = (tb / ntx) * 32, o0 = (tb % ntx) * 32;
        // load the T block in its storage order (row-major [w0][w1]), coalesced along w1
        for (int y = ty; y < 32; y += 8) {
            int a, b;   // storage coordinates (row, col) of tile element (y, tx)
            if (qc == 0) { a = i0 + y; b = o0 + tx; }   // T[i][o]
            else { a = o0 + y; b = i0 + tx; }           // T[o][i]
            tile[y][tx] = (a < w0 && b < w1) ? Tr[uint64_t(a) * w1 + b] : 0;
        }
        __syncthreads();
        for (int y = ty; y < 32; y += 8) {
            const int i = i0 + y, o = o0 + tx;
            if (i >= wi || o >= wo) continue;
            const int64_t v = qc == 0 ? tile[y][tx] : tile[tx][y];
            const uint64_t av = uabs(v);
            const uint64_t c = uint64_t(i) * wo + o;
            for (int k = 0; k < md.K; ++k) {
                uint64_t rv = mm_red(av, md.m[k], md.mu[k]);
                if (v < 0 && rv) rv = md.m[k] - rv;
                Rc[(uint64_t(k) * d + r) * cells + c] = (uint32_t)rv;
            }
        }
        __syncthreads();
    }
}

// chain mat-vec from precomputed residues: grid (row, 32-output tile, group of 8 moduli);
// 16 slices of the child index per block, combined in shared memory.
constexpr int MR_SL = 16;
__global__ void __launch_bounds__(512) k_node_matvec_r(const __grid_constant__ Node n, const __grid_constant__ Mods md,
                                                       int qc, const uint32_t *Rc, int G, uint64_t *root_part) {
    __shared__ uint64_t part[MR_SL][MV_G][MV_OUT];
    const int r = blockIdx.x;
    const int qp = 1 - qc;
    const int wi = n.w[qc], wo = n.w[qp];
    const int lane = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int o = blockIdx.y * MV_OUT + lane;
    const int g0 = blockIdx.z * G;   // G <= MV_G moduli per CTA
    const int ng = min(G, md.K - g0);
    const uint64_t cells = uint64_t(wi) * wo;
    const int chunk = (wi + MR_SL - 1) / MR_SL;
    const int i0 = sl * chunk, i1 = min(wi, i0 + chunk);
    uint64_t acc[MV_G];
#pragma unroll
    for (int g = 0; g < MV_G; ++g) acc[g] = 0;
    if (o < wo) {
#pragma unroll
        for (int g = 0; g < MV_G; ++g) {
            if (g >= ng) break;
            const int k = g0 + g;
            const uint32_t *R = Rc + (uint64_t(k) * n.d + r) * cells + o;
            const unsigned long long *x = reinterpret_cast<const unsigned long long *>(msg_row(n, qc, k, r, 0, 0));
            uint64_t a = 0;
            for (int i = i0; i < i1; ++i) a += (uint64_t)__ldg(R + uint64_t(i) * wo) * __ldg(x + i);
            acc[g] = a;   // <= chunk products of 52 bits: exact
        }
    }
#pragma unroll
    for (int g = 0; g < MV_G; ++g) part[sl][g][lane] = g < ng ? mm_red(acc[g], md.m[g0 + g], md.mu[g0 + g]) : 0;
    __syncthreads();
    if (!root_part && sl < ng && o < wo) {
        const int k = g0 + sl;
        uint64_t t = 0;
        for (int s2 = 0; s2 < MR_SL; ++s2) t = mm_add(t, part[s2][sl][lane], md.m[k]);
        const int oo = n.out_perm ? n.out_perm[uint64_t(r) * wo + o] : o;
        n.out[(uint64_t(k) * n.d + r) * n.out_bm * wo + oo] = t;
    }
    if (root_part && sl < ng) {
        // root matrix with two child legs: sum_o x_o (M y)_o, this CTA's 32 outputs reduced
        // by warp sl for modulus g0 + sl into the root partial of its output tile
        const int k = g0 + sl;
        const uint64_t m = md.m[k], mu = md.mu[k];
        uint64_t v = 0;
        if (o < wo) {
            uint64_t t = 0;
            for (int s2 = 0; s2 < MR_SL; ++s2) t = mm_add(t, part[s2][sl][lane], m);
            v = mm_mul(t, msg_row(n, qp, k, r, 0, 0)[o], m, mu);
        }
        for (int off = 16; off > 0; off >>= 1) v = mm_add(v, __shfl_xor_sync(0xffffffffu, v, off), m);
        if (lane == 0) root_part[(uint64_t(k) * n.d + r) * gridDim.y + blockIdx.y] = v;
    }
}

// acc[k][r] += sum over slots of part[k][r][slot]
__global__ void k_root_reduce(const uint64_t *part, uint64_t *acc, int slots, int d, const __grid_constant__ Mods md) {
    __shared__ uint64_t red[32];
    const int k = blockIdx.x / d;
    const uint64_t m = md.m[k];
    uint64_t s = 0;
    for (int i = threadIdx.x; i < slots; i += blockDim.x) s = mm_add(s, part[uint64_t(blockIdx.x) * slots + i], m);
    const uint64_t t = block_sum_mod(s, m, red);
    if (threadIdx.x == 0) acc[blockIdx.x] = mm_add(acc[blockIdx.x], t, m);
}

// ---------------------------------------------------------------- two-way estimate (A9)
// E_r = sum_j A[r][j] * B[r][j] in exact int128:
// |A[r][j] B[r][j]| <= N_A N_B < 2^126 for any pair of sketches built from < 2^63 tuples.
// Counter buffers are caller-owned (merged, all-reduced, or written by the caller), so the
// kernel does not rely on that: it also accumulates U = sum_j |A'_j| |B'_j| (unsigned, carry
// detected) and flags the row if a fold overflows int64 or U >= 2^127; a flagged plan is
// re-evaluated by the CRT engine (exact for any int64 counters).  Both legs are folded to
// the common width w inline (O5): A'[j] = sum_s A[j + s w].
struct DotItem {
    const int64_t *a, *b;
    uint32_t wa, wb, w;
};
constexpr int kMaxDot = 64;
struct DotItems { DotItem it[kMaxDot]; int n, d; };

__device__ __forceinline__ void add128(uint64_t &lo, uint64_t &hi, uint64_t l2, uint64_t h2) {
    const uint64_t t = lo + l2;
    hi += h2 + (t < lo);
    lo = t;
}

// one CTA per (item, row): out[(item*d + r)*3 + {0,1}] = {lo, hi} of the two's-complement
// sum, out[... + 2] = 1 if the row is flagged (not provably exact in int128), else 0
__device__ __forceinline__ bool fold_add(int64_t &x, int64_t v) {
    const int64_t t = (int64_t)((uint64_t)x + (uint64_t)v);
    const bool ovf = ((x ^ t) & (v ^ t)) < 0;
    x = t;
    return ovf;
}
__device__ __forceinline__ bool uadd128(uint64_t &lo, uint64_t &hi, uint64_t l2, uint64_t h2) {
    const uint64_t t = lo + l2;
    const uint64_t c = t < lo;
    const uint64_t h = hi + h2;
    const bool ovf = h < hi || h + c < h;
    hi = h + c;
    lo = t;
    return ovf;
}
__global__ void __launch_bounds__(512) k_dot128(const __grid_constant__ DotItems items, uint64_t *out) {
    const int item = blockIdx.x / items.d, r = blockIdx.x % items.d;
    const DotItem it = items.it[item];
    const int64_t *A = it.a + uint64_t(r) * it.wa, *B = it.b + uint64_t(r) * it.wb;
    uint64_t lo = 0, hi = 0, ulo = 0, uhi = 0;
    bool bad = false;
    for (uint32_t j = threadIdx.x; j < it.w; j += blockDim.x) {
        int64_t x = 0, y = 0;
        for (uint32_t s = j; s < it.wa; s += it.w) bad |= fold_add(x, __ldg(reinterpret_cast<const long long *>(A) + s));
        for (uint32_t s = j; s < it.wb; s += it.w) bad |= fold_add(y, __ldg(reinterpret_cast<const long long *>(B) + s));
        const __int128 p = (__int128)x * (__int128)y;
        add128(lo, hi, (uint64_t)p, (uint64_t)((unsigned __int128)p >> 64));
        const uint64_t ax = x < 0 ? 0ull - (uint64_t)x : (uint64_t)x, ay = y < 0 ? 0ull - (uint64_t)y : (uint64_t)y;
        const unsigned __int128 up = (unsigned __int128)ax * ay;
        bad |= uadd128(ulo, uhi, (uint64_t)up, (uint64_t)(up >> 64));
    }
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
        add128(lo, hi, l2, h2);
        const uint64_t u2 = __shfl_xor_sync(0xffffffffu, ulo, o), v2 = __shfl_xor_sync(0xffffffffu, uhi, o);
        bad |= uadd128(ulo, uhi, u2, v2);
    }
    bad = __any_sync(0xffffffffu, bad);
    __shared__ uint64_t slo[16], shi[16], sul[16], suh[16];
    __shared__ int sbad[16];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { slo[wid] = lo; shi[wid] = hi; sul[wid] = ulo; suh[wid] = uhi; sbad[wid] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t L = 0, H = 0, UL = 0, UH = 0;
        bool B = false;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            add128(L, H, slo[i], shi[i]);
            B |= uadd128(UL, UH, sul[i], suh[i]) || sbad[i];
        }
        B |= (UH >> 63) != 0;   // U >= 2^127: the signed sum may not fit int128
        out[uint64_t(blockIdx.x) * 3] = L;
        out[uint64_t(blockIdx.x) * 3 + 1] = H;
        out[uint64_t(blockIdx.x) * 3 + 2] = B ? 1 : 0;
    }
}

// ---------------------------------------------------------------- exact join size (accuracy evaluation)
// Frequency-vector message passing modulo one prime per blockIdx.y:
// messages [K][dom] hold lazily summed residues (< 2^26 each, so 2^38 additions fit in 64
// bits) and are reduced once after the node's pass.
constexpr int kXCols = 8, kXPreds = 8, kXChild = 4;
struct XPred { uint32_t col, kind; int64_t lo, hi; const int64_t *set; uint32_t n; };
struct XChild { const uint64_t *msg; uint32_t col; int64_t lo; uint64_t dom; };
struct XNode {
    const void *col[kXCols];
    uint32_t col64;
    uint64_t n_rows;
    uint32_t n_preds;
    XPred pred[kXPreds];
    uint32_t n_child;
    XChild ch[kXChild];
    int has_parent;
    uint32_t pcol;
    int64_t plo;
    uint64_t pdom;
    uint64_t *out;       // parent message [K][pdom], or the root's residues [K]
};
__device__ __forceinline__ int64_t xval(const XNode &n, uint32_t c, uint64_t row) {
    if ((n.col64 >> c) & 1u) return __ldg(reinterpret_cast<const long long *>(n.col[c]) + row);
    return (int64_t)__ldg(reinterpret_cast<const int *>(n.col[c]) + row);
}
__device__ __forceinline__ bool xin_set(const int64_t *s, uint32_t n, int64_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(reinterpret_cast<const long long *>(s) + mid) < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(reinterpret_cast<const long long *>(s) + lo) == v;
}
__global__ void k_exact_node(const __grid_constant__ XNode n, const __grid_constant__ Mods md, unsigned int *err) {
    __shared__ uint64_t red[32];
    const int k = blockIdx.y;
    const uint64_t m = md.m[k], mu = md.mu[k];
    uint64_t acc = 0;
    for (uint64_t row = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n.n_rows;
         row += uint64_t(gridDim.x) * blockDim.x) {
        bool ok = true;
        for (uint32_t q = 0; q < n.n_preds && ok; ++q) {
            const XPred &pr = n.pred[q];
            const int64_t v = xval(n, pr.col, row);
            if (pr.kind == SK_PRED_POINT) ok = v == pr.lo;
            else if (pr.kind == SK_PRED_RANGE) ok = pr.lo <= v && v <= pr.hi;
            else ok = xin_set(pr.set, pr.n, v);
        }
        if (!ok) continue;
        uint64_t v = 1;
        for (uint32_t c = 0; c < n.n_child; ++c) {
            const uint64_t key = (uint64_t)(xval(n, n.ch[c].col, row) - n.ch[c].lo);
            if (key >= n.ch[c].dom) { atomicOr(err, 1u); v = 0; break; }
            v = mm_mul(v, n.ch[c].msg[uint64_t(k) * n.ch[c].dom + key], m, mu);
        }
        if (n.has_parent) {
            const uint64_t key = (uint64_t)(xval(n, n.pcol, row) - n.plo);
            if (key >= n.pdom) { atomicOr(err, 1u); continue; }
            if (v) atomicAdd(reinterpret_cast<unsigned long long *>(n.out + uint64_t(k) * n.pdom + key), (unsigned long long)v);
        } else {
            acc += v;   // < 2^26 per row
        }
    }
    if (!n.has_parent) {
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) red[wid] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t t = 0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
            atomicAdd(reinterpret_cast<unsigned long long *>(n.out + k), (unsigned long long)mm_red(t, m, mu));
        }
    }
}
// msg[k][i] mod m_k
__global__ void k_mod_reduce(uint64_t *msg, uint64_t dom, const __grid_constant__ Mods md) {
    const int k = blockIdx.y;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < dom; i += uint64_t(gridDim.x) * blockDim.x)
        msg[uint64_t(k) * dom + i] = mm_red(msg[uint64_t(k) * dom + i], md.m[k], md.mu[k]);
}

// ---------------------------------------------------------------- host big integers (Garner)
struct UBig {
    std::vector<uint64_t> l;  // little-endian limbs
    void norm() { while (!l.empty() && l.back() == 0) l.pop_back(); }
    bool zero() const { return l.empty(); }
    void mul_small(uint64_t v) {
        unsigned __int128 carry = 0;
        for (auto &x : l) {
            unsigned __int128 t = (unsigned __int128)x * v + carry;
            x = (uint64_t)t;
            carry = t >> 64;
        }
        if (carry) l.push_back((uint64_t)carry);
        norm();
    }
    void add_small(uint64_t v) {
        unsigned __int128 carry = v;
        for (size_t i = 0; i < l.size() && carry; ++i) {
            unsigned __int128 t = (unsigned __int128)l[i] + carry;
            l[i] = (uint64_t)t;
            carry = t >> 64;
        }
        if (carry) l.push_back((uint64_t)carry);
    }
    static int cmp(const UBig &x, const UBig &y) {
        if (x.l.size() != y.l.size()) return x.l.size() < y.l.size() ? -1 : 1;
        for (size_t i = x.l.size(); i-- > 0;)
            if (x.l[i] != y.l[i]) return x.l[i] < y.l[i] ? -1 : 1;
        return 0;
    }
    static UBig add(const UBig &x, const UBig &y) {
        UBig r;
        r.l.resize(std::max(x.l.size(), y.l.size()) + 1, 0);
        unsigned __int128 carry = 0;
        for (size_t i = 0; i + 1 < r.l.size(); ++i) {
            const unsigned __int128 t = (unsigned __int128)(i < x.l.size() ? x.l[i] : 0) + (i < y.l.size() ? y.l[i] : 0) + carry;
            r.l[i] = (uint64_t)t;
            carry = t >> 64;
        }
        r.l.back() = (uint64_t)carry;
        r.norm();
        return r;
    }
    static UBig sub(const UBig &x, const UBig &y) {  // x >= y
        UBig r;
        r.l.resize(x.l.size());
        unsigned __int128 borrow = 0;
        for (size_t i = 0; i < x.l.size(); ++i) {
            unsigned __int128 yi = (i < y.l.size() ? y.l[i] : 0) + borrow;
            unsigned __int128 xi = x.l[i];
            if (xi >= yi) { r.l[i] = (uint64_t)(xi - yi); borrow = 0; }
            else { r.l[i] = (uint64_t)(((unsigned __int128)1 << 64) + xi - yi); borrow = 1; }
        }
        r.norm();
        return r;
    }
    int bits() const {
        if (l.empty()) return 0;
        return int(l.size() - 1) * 64 + (64 - __builtin_clzll(l.back()));
    }
    bool bit(int i) const { return (size_t)(i / 64) < l.size() && ((l[i / 64] >> (i % 64)) & 1ULL); }
    double to_double() const {  // round to nearest, ties to even
        const int nb = bits();
        if (nb == 0) return 0.0;
        if (nb <= 53) return (double)l[0];
        uint64_t top = 0;  // bits [nb-54, nb): 53 kept + 1 round bit
        for (int i = 0; i < 54; ++i)
            if (bit(nb - 54 + i)) top |= 1ULL << i;
        bool sticky = false;
        for (int i = 0; i < nb - 54 && !sticky; ++i) sticky = bit(i);
        uint64_t keep = top >> 1;
        const bool rbit = top & 1ULL;
        if (rbit && (sticky || (keep & 1ULL))) ++keep;
        return ldexp((double)keep, nb - 53);
    }
    std::string to_dec() const {
        if (l.empty()) return "0";
        UBig t = *this;
        std::string s;
        while (!t.zero()) {
            unsigned __int128 rem = 0;
            for (size_t i = t.l.size(); i-- > 0;) {
                unsigned __int128 cur = (rem << 64) | t.l[i];
                t.l[i] = (uint64_t)(cur / 10000000000000000000ULL);
                rem = cur % 10000000000000000000ULL;
            }
            t.norm();
            uint64_t r = (uint64_t)rem;
            for (int j = 0; j < 19; ++j) { s.push_back(char('0' + r % 10)); r /= 10; }
        }
        while (s.size() > 1 && s.back() == '0') s.pop_back();
        std::reverse(s.begin(), s.end());
        return s;
    }
};

struct SBig {
    bool neg = false;
    UBig mag;
    static int cmp(const SBig &x, const SBig &y) {
        const bool xz = x.mag.zero(), yz = y.mag.zero();
        const bool xn = x.neg && !xz, yn = y.neg && !yz;
        if (xn != yn) return xn ? -1 : 1;
        const int c = UBig::cmp(x.mag, y.mag);
        return xn ? -c : c;
    }
    double to_double() const { const double v = mag.to_double(); return neg ? -v : v; }
    std::string to_dec() const { return (neg && !mag.zero() ? "-" : "") + mag.to_dec(); }
};

static SBig sbig_from_i128(uint64_t lo, uint64_t hi) {
    SBig v;
    unsigned __int128 u = ((unsigned __int128)hi << 64) | lo;
    if ((int64_t)hi < 0) { v.neg = true; u = ~u + 1; }
    v.mag.l = {(uint64_t)u, (uint64_t)(u >> 64)};
    v.mag.norm();
    return v;
}

static uint64_t host_mulmod(uint64_t x, uint64_t y, uint64_t m) { return (uint64_t)((unsigned __int128)x * y % m); }
static uint64_t host_powmod(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    while (e) { if (e & 1) r = host_mulmod(r, b, m); b = host_mulmod(b, b, m); e >>= 1; }
    return r;
}
static uint64_t host_inv(uint64_t v, uint64_t m) {  // m coprime to v; extended Euclid
    __int128 t = 0, nt = 1, r = m, nr = v % m;
    while (nr) { __int128 q = r / nr; __int128 tmp = t - q * nt; t = nt; nt = tmp; tmp = r - q * nr; r = nr; nr = tmp; }
    if (t < 0) t += m;
    (void)host_powmod;
    return (uint64_t)t;
}

// Garner: residues[k] mod m_k  ->  signed integer in (-M/2, M/2]
static SBig crt_signed(const uint64_t *res, const Mods &md) {
    const int K = md.K;
    std::vector<uint64_t> v(K);
    for (int k = 0; k < K; ++k) {
        const uint64_t mk = md.m[k];
        // value of x_{<k} mod m_k and prod_{j<k} m_j mod m_k
        uint64_t xk = 0, pk = 1 % mk;
        for (int j = 0; j < k; ++j) {
            xk = (xk + host_mulmod(v[j] % mk, pk, mk)) % mk;
            pk = host_mulmod(pk, md.m[j] % mk, mk);
        }
        const uint64_t diff = (res[k] % mk + mk - xk) % mk;
        v[k] = host_mulmod(diff, host_inv(pk, mk), mk);
    }
    UBig x;
    for (int k = K - 1; k >= 0; --k) {
        x.mul_small(md.m[k]);
        x.add_small(v[k]);
    }
    UBig M;
    M.l.push_back(1);
    for (int k = 0; k < K; ++k) M.mul_small(md.m[k]);
    UBig x2 = x;
    x2.mul_small(2);
    SBig out;
    if (UBig::cmp(x2, M) > 0) { out.neg = true; out.mag = UBig::sub(M, x); }
    else out.mag = x;
    return out;
}

// ---------------------------------------------------------------- sub-plan model (host)
struct TabT {
    int t;                       // table index in the graph
    int kind;                    // KV/KM/KG
    std::vector<int> legs;       // local edge indices, canonical order
    std::vector<const sk_sketch *> sk;   // VEC/MAT: 1 sketch; MERGED: one per leg
};

struct Plan {
    std::vector<int> tabs;               // graph table indices in C (ascending)
    std::vector<int> edges;              // graph edge indices in canonical (edge-id) order
    std::vector<std::string> eid;
    std::vector<int> width;              // per local edge
    std::vector<TabT> T;
    std::vector<std::pair<int, int>> ends;   // per local edge: local table positions
    int cond = -1;
    int d = 0, device = 0;
};

static sk_status build_plan(const sk_graph *g, uint64_t mask, Plan &P) {
    if (!g) return fail(SK_EINVAL, "estimate: NULL graph");
    if (g->n_tables == 0 || g->n_tables > 64) return fail(SK_EINVAL, "estimate: n_tables must be in [1,64]");
    for (uint32_t t = 0; t < g->n_tables; ++t)
        if ((mask >> t) & 1ULL) P.tabs.push_back((int)t);
    if (P.tabs.size() < 2) return fail(SK_EINVAL, "estimate: need >= 2 tables");
    if (g->n_tables < 64 && (mask >> g->n_tables)) return fail(SK_EINVAL, "estimate: mask has bits beyond n_tables");
    std::vector<std::pair<std::string, int>> es;
    for (uint32_t e = 0; e < g->n_edges; ++e) {
        const uint32_t u = g->edge_u[e], v = g->edge_v[e];
        if (u >= g->n_tables || v >= g->n_tables || u == v) return fail(SK_EINVAL, "estimate: bad edge %u", e);
        if (((mask >> u) & 1ULL) && ((mask >> v) & 1ULL)) {
            const sk_sketch *a = g->vec_u[e], *b = g->vec_v[e];
            if (!a || !b) return fail(SK_EINVAL, "estimate: edge %u lacks a 1-D sketch", e);
            if (a->ndim != 1 || b->ndim != 1) return fail(SK_EINVAL, "estimate: edge %u sketches must be 1-D", e);
            if (a->edge[0] != b->edge[0] || a->master != b->master || a->d != b->d)
                return fail(SK_EMISMATCH, "estimate: edge %u sides disagree on id/seed/d", e);
            es.push_back({a->edge[0], (int)e});
        }
    }
    std::sort(es.begin(), es.end());
    for (size_t i = 1; i < es.size(); ++i)
        if (es[i].first == es[i - 1].first) return fail(SK_EINVAL, "estimate: duplicate edge id %s", es[i].first.c_str());
    for (auto &p : es) { P.edges.push_back(p.second); P.eid.push_back(p.first); }
    const int E = (int)P.edges.size();
    P.width.assign(E, 1 << 30);
    P.ends.assign(E, {-1, -1});
    const sk_sketch *ref = g->vec_u[P.edges.empty() ? 0 : P.edges[0]];
    if (E == 0) return fail(SK_EINVAL, "estimate: sub-plan is not connected");
    P.d = ref->d;
    P.device = ref->device;
    for (size_t i = 0; i < P.tabs.size(); ++i) {
        const int t = P.tabs[i];
        TabT tt;
        tt.t = t;
        for (int le = 0; le < E; ++le) {
            const int e = P.edges[le];
            if ((int)g->edge_u[e] == t || (int)g->edge_v[e] == t) {
                tt.legs.push_back(le);
                auto &en = P.ends[le];
                (en.first < 0 ? en.first : en.second) = (int)i;
            }
        }
        if (tt.legs.empty()) return fail(SK_EINVAL, "estimate: sub-plan is not connected");
        if (tt.legs.size() > 3) return fail(SK_EOVERFLOW, "estimate: table with >3 join edges in a sub-plan is unsupported");
        auto side = [&](int le) -> const sk_sketch * {
            const int e = P.edges[le];
            return (int)g->edge_u[e] == t ? g->vec_u[e] : g->vec_v[e];
        };
        if (tt.legs.size() == 1) {
            tt.kind = KV;
            tt.sk.push_back(side(tt.legs[0]));
        } else {
            // a built matrix (2 legs) or 3-D tensor (3 legs) over
            // exactly this table's sub-plan edges (reading R8), else the merged view
            const sk_sketch *mat = nullptr;
            for (uint32_t mi = 0; mi < g->n_mats; ++mi) {
                if ((int)g->mat_table[mi] != t || !g->mat[mi]) continue;
                const sk_sketch *ms = g->mat[mi];
                if (ms->ndim != tt.legs.size()) continue;
                bool same = true;
                for (size_t q = 0; q < tt.legs.size(); ++q) same &= ms->edge[q] == P.eid[tt.legs[q]];
                if (same) mat = ms;
            }
            if (mat) { tt.kind = mat->ndim == 3 ? KT : KM; tt.sk.push_back(mat); }
            else { tt.kind = KG; for (int le : tt.legs) tt.sk.push_back(side(le)); }
        }
        for (const sk_sketch *s : tt.sk) {
            if (s->d != P.d) return fail(SK_EMISMATCH, "estimate: sketches disagree on d");
            if (s->device != P.device) return fail(SK_EMISMATCH, "estimate: sketches on different devices");
            if (s->master != ref->master) return fail(SK_EMISMATCH, "estimate: sketches disagree on master seed");
        }
        for (size_t q = 0; q < tt.legs.size(); ++q) {
            const int wn = (tt.kind == KM || tt.kind == KT) ? (int)tt.sk[0]->w[q] : (int)tt.sk[tt.kind == KV ? 0 : q]->w[0];
            P.width[tt.legs[q]] = std::min(P.width[tt.legs[q]], wn);
        }
        P.T.push_back(tt);
    }
    // connectivity
    {
        std::vector<int> seen(P.tabs.size(), 0), st{0};
        seen[0] = 1;
        while (!st.empty()) {
            const int i = st.back(); st.pop_back();
            for (int le : P.T[i].legs) {
                const int j = P.ends[le].first == i ? P.ends[le].second : P.ends[le].first;
                if (!seen[j]) { seen[j] = 1; st.push_back(j); }
            }
        }
        for (int s : seen) if (!s) return fail(SK_EINVAL, "estimate: sub-plan is not connected");
    }
    const int cyc = E - (int)P.tabs.size() + 1;
    if (cyc > 1) return fail(SK_EOVERFLOW, "estimate: sub-plans with more than one independent cycle are unsupported");
    if (cyc == 1) {
        // condition on the cycle edge whose endpoints have the most legs (ties: canonical order)
        int best = -1, bestdeg = -1;
        for (int le = 0; le < E; ++le) {
            std::vector<int> seen(P.tabs.size(), 0), st{0};
            seen[0] = 1;
            while (!st.empty()) {
                const int i = st.back(); st.pop_back();
                for (int f : P.T[i].legs) {
                    if (f == le) continue;
                    const int j = P.ends[f].first == i ? P.ends[f].second : P.ends[f].first;
                    if (!seen[j]) { seen[j] = 1; st.push_back(j); }
                }
            }
            bool on = true;
            for (int s : seen) if (!s) on = false;
            if (!on) continue;
            const int dg = (int)P.T[P.ends[le].first].legs.size() + (int)P.T[P.ends[le].second].legs.size();
            if (dg > bestdeg) { bestdeg = dg; best = le; }
        }
        P.cond = best;
    }
    return SK_OK;
}

// stream-ordered device temporary; non-copyable (kept in a std::deque so growth never
// relocates, and therefore never frees, a live buffer)
struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { if (p) cudaFreeAsync(p, s); }
};
using DevPool = std::deque<DevBuf>;

static sk_status dalloc(DevPool &pool, size_t bytes, cudaStream_t s, void **out) {
    pool.emplace_back();
    pool.back().s = s;
    cudaError_t e = cudaMallocAsync(&pool.back().p, std::max<size_t>(bytes, 16), s);
    if (e != cudaSuccess) { pool.back().p = nullptr; return cuda_fail(e, "cudaMallocAsync(estimate)"); }
    *out = pool.back().p;
    return SK_OK;
}

static Mods mods_for(double logB, int K_min) {
    Mods md;
    md.K = 0;
    double have = 0;
    while (md.K < kMaxMod && (have < logB * (1 + 1e-9) + 3.0 || md.K < K_min)) {
        md.m[md.K] = kPrimes[md.K];
        md.mu[md.K] = (uint64_t)(((unsigned __int128)1 << 64) / kPrimes[md.K]);
        have += log2((double)kPrimes[md.K]) - 1e-9;
        ++md.K;
    }
    return md;
}

static double mods_capacity(const Mods &md) {
    double have = 0;
    for (int k = 0; k < md.K; ++k) have += log2((double)md.m[k]) - 1e-9;
    return have;
}

// log2 of a rigorous bound on |E_r| from per-sketch L1 values, the smaller of
//  (a) prod_t ||T_t||_1 (every term of the expansion is one choice of an entry per tensor),
//      a merged view's L1 taken as its best constituent's times the other legs' widths;
//  (b) prod_t F_t, F_t = ||T_t||_1 for vectors and matrices and max_q ||v_q||_1 for a merged
//      view: in message passing a node's output L1 is at most (sum over its parent leg of
//      |entries| <= F_t) times its children's message L1s, and a root's value at most
//      max|entry| <= F_t times them, since |min-abs(v_1, ..)| <= |v_q| for every constituent;
//      a conditioned cycle adds the factor w of the conditioned edge (sum over its buckets).
template <typename F>
static double log_bound(const Plan &P, F l1of) {
    double a = 0, b = 0;
    bool has_kg = false;
    for (auto &t : P.T) {
        if (t.kind != KG) {
            const double v = log2(std::max(1.0, l1of(t.sk[0])));
            a += v;
            b += v;
            continue;
        }
        has_kg = true;
        double best = 1e300, mx = 0;
        for (size_t q = 0; q < t.legs.size(); ++q) {
            const double l = log2(std::max(1.0, l1of(t.sk[q])));
            double v = l;
            for (size_t q2 = 0; q2 < t.legs.size(); ++q2) if (q2 != q) v += log2((double)P.width[t.legs[q2]]);
            best = std::min(best, v);
            mx = std::max(mx, l);
        }
        a += best;
        b += mx;
    }
    if (P.cond >= 0 && has_kg) b += log2((double)P.width[P.cond]);
    return std::min(a, b);
}

// Spanning tree of a plan rooted at local table 0 without the conditioned edge: parent edge
// per table (-1 at the root) and a post-order for message passing.
static void spanning_tree(const Plan &P, std::vector<int> &parent_edge, std::vector<int> &order) {
    const int NT = (int)P.T.size();
    parent_edge.assign(NT, -2);
    std::vector<std::pair<int, int>> st2{{0, -1}};
    std::vector<int> vis(NT, 0), pre;
    while (!st2.empty()) {
        auto [i, pe] = st2.back();
        st2.pop_back();
        if (vis[i]) continue;
        vis[i] = 1;
        parent_edge[i] = pe;
        pre.push_back(i);
        for (int le : P.T[i].legs) {
            if (le == pe || le == P.cond) continue;
            const int j = P.ends[le].first == i ? P.ends[le].second : P.ends[le].first;
            if (!vis[j]) st2.push_back({j, le});
        }
    }
    order.assign(pre.rbegin(), pre.rend());
}

// log2 bound of each node's output (message, per conditioned bucket; the root's value) in
// message passing: F_t x the bounds of its children's messages (see log_bound (b)).
// logF: per local table.  A merged node whose bound is <= 61 runs in 64-bit arithmetic.
static void node_logbounds(const Plan &P, const std::vector<double> &logF, std::vector<double> &lb) {
    std::vector<int> parent_edge, order;
    spanning_tree(P, parent_edge, order);
    const int NT = (int)P.T.size();
    lb.assign(NT, 0.0);
    for (int i : order) {
        double v = logF[i];
        for (int le : P.T[i].legs) {
            if (le == parent_edge[i] || le == P.cond) continue;
            const int j = P.ends[le].first == i ? P.ends[le].second : P.ends[le].first;
            v += lb[j];
        }
        lb[i] = v;
    }
}

// Residues (and tensor-core M planes) of matrices per (matrix pointer, orientation): computed
// once per batch, or once per planning call for the sketches' own counters (BatchShare: their
// contents cannot change while plan_greedy / plan_enumerate runs; one map per modulus count)
using ResKey = std::pair<const void *, int>;
struct BatchShare {
    DevPool pool;
    std::map<int, std::map<ResKey, uint32_t *>> by_K;
    std::set<const void *> stable;
    std::map<const sk_sketch *, std::vector<uint64_t>> l1;   // per-row L1 norms (host)
    explicit BatchShare(const sk_graph *g) {
        if (!g) return;
        for (uint32_t m = 0; m < g->n_mats; ++m)
            if (g->mat && g->mat[m]) stable.insert(g->mat[m]->counters);
    }
};
struct ResCache {
    std::map<ResKey, uint32_t *> map;
    std::map<ResKey, uint32_t *> *shared = nullptr;
    DevPool *spool = nullptr;
    const std::set<const void *> *stable = nullptr;
    bool is_shared(const void *p) const { return shared && stable && stable->count(p); }
    uint32_t *find(const ResKey &k) const {
        const auto &m = is_shared(k.first) ? *shared : map;
        auto it = m.find(k);
        return it == m.end() ? nullptr : it->second;
    }
    void put(const ResKey &k, uint32_t *p) { (is_shared(k.first) ? *shared : map)[k] = p; }
    DevPool &pool_for(const void *p, DevPool &batch) { return is_shared(p) ? *spool : batch; }
};

// Enqueue every kernel of one sub-plan on `stream` (no host synchronisation): per-row
// residues -> acc[K][d] (zeroed by the caller), per-sketch-row L1 norms -> l1[n_uniq][d].
static sk_status enqueue_plan(const Plan &P, const Mods &md, std::vector<const sk_sketch *> &uniq,
                              DevPool &pool, uint64_t *acc, unsigned long long *l1, cudaStream_t stream,
                              int ring = 0, ResCache *rescache = nullptr,
                              const Mods *resmods = nullptr, const std::vector<char> *narrow = nullptr,
                              std::map<std::tuple<const void *, int, int>, const int64_t *> *foldcache = nullptr,
                              std::map<std::pair<const void *, int>, std::array<void *, 4>> *sortcache = nullptr,
                              std::map<std::vector<const void *>, std::array<const uint32_t *, 3>> *rankcache = nullptr) {
    // ring: 0 = CRT residues, 1 = exact int128, 2 = fp64 absolute-value bound (no matrices)
    const bool exact = ring == 1, absb = ring == 2;
    const int E = (int)P.edges.size();
    const int NT = (int)P.T.size();
    const int d = P.d;
    const int K = exact ? 2 : absb ? 1 : md.K;   // 64-bit words per message entry and row
    sk_status st;
    // ---- L1 norms of every sketch involved (checked against the moduli after the batch;
    //      skipped when the caller computes them once for the whole batch: l1 == null)
    for (size_t b0 = 0; l1 && b0 < uniq.size(); b0 += kMaxL1Items) {
        L1Items items;
        items.n = (int)std::min<size_t>(kMaxL1Items, uniq.size() - b0);
        uint32_t maxcells = 1;
        for (int i = 0; i < items.n; ++i) {
            const sk_sketch *s = uniq[b0 + i];
            items.it[i] = {s->counters, s->d, (uint32_t)(s->n_counters / s->d)};
            maxcells = std::max(maxcells, items.it[i].cells);
        }
        const unsigned chunks = std::min<unsigned>(64, (maxcells + 8191) / 8192);
        k_l1<<<dim3(items.n, d, chunks), 256, 0, stream>>>(items, l1 + b0 * d, d); count_launch();
        SKB_CUDA_CHECK("estimate launch 1");
    }
    // ---- folded copies of every tensor leg
    std::vector<std::vector<const int64_t *>> data(NT);
    for (int i = 0; i < NT; ++i) {
        const TabT &t = P.T[i];
        if (t.kind == KT) {
            const sk_sketch *s = t.sk[0];
            const int w0 = P.width[t.legs[0]], w1 = P.width[t.legs[1]], w2 = P.width[t.legs[2]];
            if ((int)s->w[0] == w0 && (int)s->w[1] == w1 && (int)s->w[2] == w2) { data[i].push_back(s->counters); continue; }
            void *f;
            if ((st = dalloc(pool, size_t(d) * w0 * w1 * w2 * 8, stream, &f))) return st;
            k_fold3<<<1184, 256, 0, stream>>>(s->counters, (int64_t *)f, d, s->w[0], s->w[1], s->w[2], w0, w1, w2);
            count_launch();
            data[i].push_back((const int64_t *)f);
        } else if (t.kind == KM) {
            const sk_sketch *s = t.sk[0];
            const int w0 = P.width[t.legs[0]], w1 = P.width[t.legs[1]];
            if ((int)s->w[0] == w0 && (int)s->w[1] == w1) { data[i].push_back(s->counters); continue; }
            const auto key = std::make_tuple((const void *)s, w0, w1);
            if (foldcache && foldcache->count(key)) { data[i].push_back((*foldcache)[key]); continue; }
            void *f;
            if ((st = dalloc(pool, size_t(d) * w0 * w1 * 8, stream, &f))) return st;
            k_fold<<<1184, 256, 0, stream>>>(s->counters, (int64_t *)f, d, s->w[0], s->w[1], w0, w1); count_launch();
            data[i].push_back((const int64_t *)f);
            if (foldcache) (*foldcache)[key] = (const int64_t *)f;
        } else {
            for (size_t q = 0; q < t.sk.size(); ++q) {
                const sk_sketch *s = t.sk[q];
                const int w = P.width[t.legs[q]];
                if ((int)s->w[0] == w) { data[i].push_back(s->counters); continue; }
                const auto key = std::make_tuple((const void *)s, 1, w);
                if (foldcache && foldcache->count(key)) { data[i].push_back((*foldcache)[key]); continue; }
                void *f;
                if ((st = dalloc(pool, size_t(d) * w * 8, stream, &f))) return st;
                k_fold<<<592, 256, 0, stream>>>(s->counters, (int64_t *)f, d, 1, s->w[0], 1, w); count_launch();
                data[i].push_back((const int64_t *)f);
                if (foldcache) (*foldcache)[key] = (const int64_t *)f;
            }
        }
    }
    SKB_CUDA_CHECK("estimate launch 2");
    // ---- spanning tree rooted at local table 0 (DFS), post-order
    std::vector<int> parent_edge, order;
    spanning_tree(P, parent_edge, order);
    // does the subtree of node i contain an endpoint of the conditioned edge?
    std::vector<int> depb(NT, 0);
    for (int i : order) {
        if (P.cond >= 0 && (P.ends[P.cond].first == i || P.ends[P.cond].second == i)) depb[i] = 1;
        for (int le : P.T[i].legs) {
            if (le == parent_edge[i] || le == P.cond) continue;
            const int j = P.ends[le].first == i ? P.ends[le].second : P.ends[le].first;
            if (depb[j]) depb[i] = 1;
        }
    }
    // ---- sorted orders for merged nodes' contracted legs
    std::vector<int> qc_of(NT, -1);
    std::vector<const uint32_t *> pos_of(NT, nullptr);   // exact merged nodes: precomputed thresholds
    std::vector<const int32_t *> ord_of(NT, nullptr);
    std::vector<const uint64_t *> sabs_of(NT, nullptr);
    std::vector<const int64_t *> csorted_of(NT, nullptr);
    std::vector<std::array<const uint32_t *, 3>> rank_of(NT, {nullptr, nullptr, nullptr});
    std::vector<const int32_t *> perm_of_edge(E, nullptr);   // messages delivered in the parent's sorted order
    for (int i = 0; i < NT; ++i) {
        const TabT &t = P.T[i];
        if (t.kind != KG) continue;
        int qc = -1;
        for (size_t q = 0; q < t.legs.size(); ++q) {
            const int le = t.legs[q];
            if (le == parent_edge[i] || le == P.cond) continue;
            qc = (int)q;
            break;
        }
        if (qc < 0) continue;   // merged leaf: evaluated densely
        const int w = P.width[t.legs[qc]];
        if (w > 8192) return fail(SK_EOVERFLOW, "estimate: merged contraction supports widths <= 8192");
        void *o, *sa, *rk, *csd;
        const auto skey = std::make_pair((const void *)data[i][qc], w);
        if (sortcache && sortcache->count(skey)) {   // this constituent was sorted for an earlier plan of the batch
            const auto &c = (*sortcache)[skey];
            o = c[0]; sa = c[1]; rk = c[2]; csd = c[3];
        } else {
            if ((st = dalloc(pool, size_t(d) * w * 4, stream, &o))) return st;
            if ((st = dalloc(pool, size_t(d) * w * 8, stream, &sa))) return st;
            if ((st = dalloc(pool, size_t(d) * w * 4, stream, &rk))) return st;
            if ((st = dalloc(pool, size_t(d) * w * 8, stream, &csd))) return st;
            const size_t sm = size_t(w) * 12;
            SKB_CUDA(cudaFuncSetAttribute(k_sort_abs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_sort_abs<<<d, 512, sm, stream>>>(data[i][qc], w, (int32_t *)o, (uint64_t *)sa, (int32_t *)rk, (int64_t *)csd); count_launch();
            if (sortcache) (*sortcache)[skey] = {o, sa, rk, csd};
        }
        perm_of_edge[t.legs[qc]] = (const int32_t *)rk;
        csorted_of[i] = (const int64_t *)csd;
        SKB_CUDA_CHECK("estimate launch 3");
        qc_of[i] = qc;
        ord_of[i] = (const int32_t *)o;
        sabs_of[i] = (const uint64_t *)sa;
        if (absb || getenv("COMPASS_EST_NO_RANK")) continue;
        // ranks of every other leg's constituent values in this sorted order (thresholds of the
        // O9 identity by lookup instead of a binary search per output)
        Node rn;
        memset(&rn, 0, sizeof(rn));
        rn.nl = (int)t.legs.size();
        rn.qc = qc;
        rn.sabs = sabs_of[i];
        uint32_t *ro[3] = {nullptr, nullptr, nullptr};
        int wmax = 1;
        std::vector<const void *> rkey{(const void *)(intptr_t)qc};
        for (int q = 0; q < rn.nl; ++q) {
            rn.w[q] = P.width[t.legs[q]];
            rn.data[q] = data[i][q];
            rkey.push_back(data[i][q]);
            rkey.push_back((const void *)(intptr_t)rn.w[q]);
        }
        if (sortcache && rankcache && rankcache->count(rkey)) {   // same merged view, same contracted leg
            const auto &c = (*rankcache)[rkey];
            for (int q = 0; q < 3; ++q) rank_of[i][q] = c[q];
            continue;
        }
        for (int q = 0; q < rn.nl; ++q) {
            if (q == qc) continue;
            void *rb;
            if ((st = dalloc(pool, size_t(d) * rn.w[q] * 4, stream, &rb))) return st;
            ro[q] = (uint32_t *)rb;
            wmax = std::max(wmax, rn.w[q]);
        }
        k_merged_rank<<<dim3((wmax + 255) / 256, d), 256, 0, stream>>>(rn, ro[0], ro[1], ro[2]); count_launch();
        for (int q = 0; q < 3; ++q) rank_of[i][q] = ro[q];
        if (sortcache && rankcache) (*rankcache)[rkey] = {ro[0], ro[1], ro[2]};
    }
    // ---- chunking of the conditioned bucket
    const int64_t Btot = P.cond >= 0 ? P.width[P.cond] : 1;
    size_t per_b = size_t(K) * d * 8;                      // root partials
    for (int i : order)
        if (parent_edge[i] >= 0 && depb[i]) per_b += size_t(K) * d * P.width[parent_edge[i]] * 8;
    int64_t Bc = Btot;
    while (Bc > 1 && per_b * Bc > (size_t(3) << 30)) Bc = (Bc + 1) / 2;
    // message buffers per local edge
    std::vector<uint64_t *> msg(E, nullptr);
    std::vector<int> msg_bm(E, 1);
    std::vector<char> msg64(E, 0);   // exact engine: the edge's message is stored as int64
    for (int i : order) {
        const int pe = parent_edge[i];
        if (pe < 0) continue;
        msg_bm[pe] = depb[i] ? (int)Bc : 1;
        void *mb;
        if ((st = dalloc(pool, size_t(K) * d * msg_bm[pe] * P.width[pe] * 8, stream, &mb))) return st;
        msg[pe] = (uint64_t *)mb;
    }
    const int tiles_root = 1;
    void *part;
    if ((st = dalloc(pool, size_t(K) * d * Bc * tiles_root * 8, stream, &part))) return st;
    for (int64_t b0 = 0; b0 < Btot; b0 += Bc) {
        const int B = (int)std::min<int64_t>(Bc, Btot - b0);
        uint64_t *dense_root_part = nullptr;   // modular dense root split over tiles
        int dense_root_slots = 0;
        for (int i : order) {
            const TabT &t = P.T[i];
            const int pe = parent_edge[i];
            Node n;
            memset(&n, 0, sizeof(n));
            n.kind = t.kind;
            n.nl = (int)t.legs.size();
            n.d = d;
            n.B = B;
            n.b0 = b0;
            for (int q = 0; q < n.nl; ++q) {
                const int le = t.legs[q];
                n.w[q] = P.width[le];
                n.role[q] = (le == P.cond) ? RFIXED : (le == pe ? RPARENT : RCHILD);
                if (n.role[q] == RCHILD) {
                    n.msg[q] = msg[le];
                    n.bm[q] = msg_bm[le];
                    if (msg64[le]) n.m64 |= 1 << q;
                }
                n.data[q] = (t.kind == KG) ? data[i][q] : data[i][0];
            }
            // nodes whose message does not depend on b are computed once (first chunk)
            if (pe >= 0 && msg_bm[pe] == 1 && b0 > 0) continue;
            const int nB = (pe >= 0 && msg_bm[pe] == 1) ? 1 : B;
            n.B = nB;
            int tiles = 1;
            const int blocks_xy = K * d * nB;
            if (pe >= 0) {
                n.out = msg[pe];
                n.out_bm = msg_bm[pe];
                n.out_perm = perm_of_edge[pe];
                const int wo = P.width[pe];
                while (blocks_xy * tiles < 592 && tiles * 256 < wo) tiles *= 2;
            } else {
                n.out = (uint64_t *)part;
            }
            n.tiles = tiles;
            int nchild = 0, qchild = -1;
            bool hasfixed = false;
            for (int q = 0; q < n.nl; ++q) {
                if (n.role[q] == RCHILD) { ++nchild; qchild = q; }
                if (n.role[q] == RFIXED) hasfixed = true;
            }
            if (absb) {
                if (t.kind == KG && qc_of[i] >= 0) {
                    n.qc = qc_of[i];
                    n.ord = ord_of[i];
                    n.sabs = sabs_of[i];
                    n.csorted = csorted_of[i];
                    for (int q = 0; q < 3; ++q) n.rank[q] = rank_of[i][q];
                    int wo_max = 1;
                    for (int q = 0; q < n.nl; ++q)
                        if (q != n.qc && n.role[q] != RFIXED) wo_max = std::max(wo_max, n.w[q]);
                    int mtiles = 1;
                    while (d * nB * mtiles < 296 && mtiles * MX_T < wo_max) mtiles *= 2;
                    n.tiles = (pe >= 0) ? mtiles : 1;
                    const size_t sm = size_t(2) * (n.w[n.qc] + 1) * 8;
                    SKB_CUDA(cudaFuncSetAttribute(k_node_merged_abs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                    k_node_merged_abs<<<dim3(d * nB, n.tiles), MX_T, sm, stream>>>(n); count_launch();
                } else {
                    int xt = 1;
                    if (pe >= 0) while (d * nB * xt < 592 && xt * 256 < P.width[pe]) xt *= 2;
                    n.tiles = (pe >= 0) ? xt : 1;
                    k_node_dense_abs<<<dim3(d * nB, n.tiles), 256, 0, stream>>>(n); count_launch();
                }
            } else if (exact) {
                if (t.kind == KG && qc_of[i] >= 0) {
                    n.qc = qc_of[i];
                    n.ord = ord_of[i];
                    n.sabs = sabs_of[i];
                    n.csorted = csorted_of[i];
                    for (int q = 0; q < 3; ++q) n.rank[q] = rank_of[i][q];
                    // outer leg: the parent, else the first other child (as in the kernel)
                    int wo_max = 1, qo = -1, nother = 0;
                    bool fixed = false;
                    for (int q = 0; q < n.nl; ++q) {
                        if (q == n.qc) continue;
                        if (n.role[q] == RFIXED) { fixed = true; continue; }
                        wo_max = std::max(wo_max, n.w[q]);
                        if (qo < 0) qo = q;
                        ++nother;
                    }
                    for (int q = 0; q < n.nl; ++q) if (q != n.qc && n.role[q] == RPARENT) qo = q;
                    const uint32_t *pos = nullptr;
                    if (!fixed && nother == 1 && qo >= 0) {
                        // thresholds depend on the outer index only: once per node
                        if (!pos_of[i]) {
                            void *pb;
                            if ((st = dalloc(pool, size_t(d) * n.w[qo] * 4, stream, &pb))) return st;
                            k_merged_pos<<<dim3((n.w[qo] + 255) / 256, d), 256, 0, stream>>>(n, qo, (uint32_t *)pb); count_launch();
                            pos_of[i] = (const uint32_t *)pb;
                        }
                        pos = pos_of[i];
                    }
                    int mtiles = 1;
                    while (d * nB * mtiles < 296 && mtiles * MX_T < wo_max) mtiles *= 2;
                    n.tiles = (pe >= 0) ? mtiles : 1;
                    const bool nw = narrow && (*narrow)[i] && !getenv("COMPASS_EST_NO_NARROW");
                    if (nw && pe >= 0) { n.out64 = 1; msg64[pe] = 1; }   // |message| <= node bound <= 2^61
                    const size_t sm = size_t(2) * (n.w[n.qc] + (n.w[n.qc] >> 3) + 1) * (nw ? 8 : 16);   // padded prefixes
                    if (sm + 2 * MX_T * 16 + 1024 > 227 * 1024) return fail(SK_EOVERFLOW, "estimate: merged contraction too wide");
                    if (nw) {
                        SKB_CUDA(cudaFuncSetAttribute(k_node_merged_x<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                        k_node_merged_x<int64_t><<<dim3(d * nB, n.tiles), MX_T, sm, stream>>>(n, pos);
                    } else {
                        SKB_CUDA(cudaFuncSetAttribute(k_node_merged_x<i128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                        k_node_merged_x<i128><<<dim3(d * nB, n.tiles), MX_T, sm, stream>>>(n, pos);
                    }
                    count_launch();
                } else {
                    int xt = 1;
                    if (pe >= 0) while (d * nB * xt < 592 && xt * 256 < P.width[pe]) xt *= 2;
                    n.tiles = (pe >= 0) ? xt : 1;
                    k_node_dense_x<<<dim3(d * nB, n.tiles), 256, 0, stream>>>(n); count_launch();
                }
            } else if (t.kind == KM && pe >= 0 && nchild == 1 && !hasfixed && nB == 1 && rescache && resmods && !getenv("COMPASS_EST_NO_RES") &&
                       md.K <= resmods->K && !getenv("COMPASS_EST_NO_MATVEC")) {
                // residues of this (folded) matrix in this orientation: once per batch
                const auto key = std::make_pair((const void *)n.data[0], qchild);
                uint32_t *Rc = rescache->find(key);
                if (!Rc) {
                    void *rb;
                    const size_t cells = size_t(n.w[0]) * n.w[1];
                    if ((st = dalloc(rescache->pool_for(key.first, pool), size_t(resmods->K) * d * cells * 4, stream, &rb))) return st;
                    k_mat_residues<<<dim3(std::max(1, 1184 / d), 1, d), 256, 0, stream>>>(n.data[0], d, n.w[0], n.w[1], qchild, *resmods, (uint32_t *)rb);
                    count_launch();
                    Rc = (uint32_t *)rb;
                    rescache->put(key, Rc);
                }
                // one modulus per CTA unless that makes the grid very large (more CTAs in
                // flight hide the latency of the residue loads)
                const int nto = (P.width[pe] + MV_OUT - 1) / MV_OUT;
                const int G = (d * nto * md.K <= 4096) ? 1 : MV_G;
                k_node_matvec_r<<<dim3(d, nto, (md.K + G - 1) / G), 512, 0, stream>>>(n, md, qchild, Rc, G, nullptr);
                count_launch();
            } else if (t.kind == KM && pe < 0 && nchild == 2 && !hasfixed && nB == 1 && rescache && resmods &&
                       !getenv("COMPASS_EST_NO_RES") && md.K <= resmods->K && !getenv("COMPASS_EST_NO_MATVEC")) {
                // root matrix with two child legs: the mat-vec over leg 1 (residues cached per
                // batch), dotted with the leg-0 message inside the same kernel
                const int qc = 1, qo = 0;
                const auto key = std::make_pair((const void *)n.data[0], qc);
                uint32_t *Rc = rescache->find(key);
                if (!Rc) {
                    void *rb;
                    const size_t cells = size_t(n.w[0]) * n.w[1];
                    if ((st = dalloc(rescache->pool_for(key.first, pool), size_t(resmods->K) * d * cells * 4, stream, &rb))) return st;
                    k_mat_residues<<<dim3(std::max(1, 1184 / d), 1, d), 256, 0, stream>>>(n.data[0], d, n.w[0], n.w[1], qc, *resmods, (uint32_t *)rb);
                    count_launch();
                    Rc = (uint32_t *)rb;
                    rescache->put(key, Rc);
                }
                const int nto = (n.w[qo] + MV_OUT - 1) / MV_OUT;
                const int G = (d * nto * md.K <= 4096) ? 1 : MV_G;
                void *pr;
                if ((st = dalloc(pool, size_t(K) * d * nto * 8, stream, &pr))) return st;
                k_node_matvec_r<<<dim3(d, nto, (md.K + G - 1) / G), 512, 0, stream>>>(n, md, qc, Rc, G, (uint64_t *)pr);
                count_launch();
                dense_root_part = (uint64_t *)pr;
                dense_root_slots = nto;
            } else if (t.kind == KM && pe >= 0 && nchild == 1 && !hasfixed && nB == 1 && !getenv("COMPASS_EST_NO_MATVEC")) {
                k_node_matvec<<<dim3(d, (P.width[pe] + MV_OUT - 1) / MV_OUT), 256, 0, stream>>>(n, md, qchild); count_launch();
            } else if (t.kind == KM && pe >= 0 && nchild == 1 && !hasfixed && nB >= 16) {
                const int nbt = (nB + GBM - 1) / GBM;
                const int njt = (P.width[pe] + GBN - 1) / GBN;
                const uint32_t *Rc = nullptr;   // residues shared with the chain mat-vecs of the batch
                if (rescache && resmods && md.K <= resmods->K) {
                    const auto key = std::make_pair((const void *)n.data[0], qchild);
                    Rc = rescache->find(key);
                    if (!Rc) {
                        void *rb;
                        const size_t cells = size_t(n.w[0]) * n.w[1];
                        if ((st = dalloc(rescache->pool_for(key.first, pool), size_t(resmods->K) * d * cells * 4, stream, &rb))) return st;
                        k_mat_residues<<<dim3(std::max(1, 1184 / d), 1, d), 256, 0, stream>>>(n.data[0], d, n.w[0], n.w[1], qchild, *resmods, (uint32_t *)rb);
                        count_launch();
                        rescache->put(key, (uint32_t *)rb);
                        Rc = (uint32_t *)rb;
                    }
                }
                const char *ge = getenv("COMPASS_GEMM");
                if (Rc && n.w[qchild] <= 8192 && !(ge && (strcmp(ge, "cuda") == 0 || strcmp(ge, "tc") == 0))) {
                    // tensor cores fed by bulk copies of pre-tiled byte planes: x planes per
                    // node, M planes cached per batch with the residues
                    const int wi = n.w[qchild], wj = P.width[pe];
                    const int tbt = (nB + TC_M - 1) / TC_M, tjt = (wj + TC_N - 1) / TC_N, tkb = (wi + TC_KB - 1) / TC_KB;
                    const int Kres = resmods->K;
                    const auto pkey = std::make_pair((const void *)n.data[0], qchild + 16);
                    unsigned char *Mp = (unsigned char *)rescache->find(pkey);
                    if (!Mp) {
                        void *pm;
                        if ((st = dalloc(rescache->pool_for(pkey.first, pool), size_t(Kres) * d * tjt * tkb * (4 * TC_B_PLANE), stream, &pm))) return st;
                        k_planes_m<<<1184, 256, 0, stream>>>(Rc, Kres * d, wi, wj, tjt, tkb, (unsigned char *)pm);
                        count_launch();
                        rescache->put(pkey, (uint32_t *)pm);
                        Mp = (unsigned char *)pm;
                    }
                    void *px;
                    if ((st = dalloc(pool, size_t(K) * d * tbt * tkb * (4 * TC_A_PLANE), stream, &px))) return st;
                    k_planes_x<<<1184, 256, 0, stream>>>(n, qchild, K, tbt, tkb, (unsigned char *)px);
                    count_launch();
                    static bool attr2 = false;
                    if (!attr2) {
                        SKB_CUDA(cudaFuncSetAttribute(k_node_mat_gemm_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM2));
                        attr2 = true;
                    }
                    if (getenv("COMPASS_EST_DEBUG"))
                        fprintf(stderr, "gemm tc bulk: K %d d %d B %d wi %d wj %d\n", K, d, nB, wi, wj);
                    int dev_g = 0, sms_g = 148;
                    cudaGetDevice(&dev_g);
                    cudaDeviceGetAttribute(&sms_g, cudaDevAttrMultiProcessorCount, dev_g);
                    const int ntl = K * d * tbt * tjt;
                    k_node_mat_gemm_bulk<<<std::min(ntl, sms_g), 192, TC_SMEM2, stream>>>(n, md, qchild, (const unsigned char *)px,
                                                                                         Mp, tbt, tjt, tkb, 0);
                } else if (Rc && n.w[qchild] <= 8192 && !(ge && strcmp(ge, "cuda") == 0)) {
                    // tensor cores (tcgen05 kind::i8 on byte planes), same residues
                    static bool attr_set = false;
                    if (!attr_set) {
                        SKB_CUDA(cudaFuncSetAttribute(k_node_mat_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
                        attr_set = true;
                    }
                    const int tbt = (nB + TC_M - 1) / TC_M, tjt = (P.width[pe] + TC_N - 1) / TC_N;
                    if (getenv("COMPASS_EST_DEBUG"))
                        fprintf(stderr, "gemm tc: K %d d %d B %d wi %d wj %d\n", K, d, nB, n.w[qchild], P.width[pe]);
                    k_node_mat_gemm_tc<<<dim3(K * d, tbt * tjt), 256, TC_SMEM, stream>>>(n, md, qchild, Rc);
                } else {
                    k_node_mat_gemm<<<dim3(K * d, nbt * njt), 256, 0, stream>>>(n, md, qchild, Rc);
                }
                count_launch();
            } else if (t.kind == KG && qc_of[i] >= 0) {
                n.qc = qc_of[i];
                n.ord = ord_of[i];
                n.sabs = sabs_of[i];
                n.csorted = csorted_of[i];
                for (int q = 0; q < 3; ++q) n.rank[q] = rank_of[i][q];
                int wo_max = 1, qo = -1, nother = 0;
                bool fixed = false;
                for (int q = 0; q < n.nl; ++q) {
                    if (q == n.qc) continue;
                    if (n.role[q] == RFIXED) { fixed = true; continue; }
                    wo_max = std::max(wo_max, n.w[q]);
                    if (qo < 0) qo = q;
                    ++nother;
                }
                for (int q = 0; q < n.nl; ++q) if (q != n.qc && n.role[q] == RPARENT) qo = q;
                const uint32_t *pos = nullptr;
                if (!fixed && nother == 1 && qo >= 0) {
                    if (!pos_of[i]) {
                        void *pb;
                        if ((st = dalloc(pool, size_t(d) * n.w[qo] * 4, stream, &pb))) return st;
                        k_merged_pos<<<dim3((n.w[qo] + 255) / 256, d), 256, 0, stream>>>(n, qo, (uint32_t *)pb); count_launch();
                        pos_of[i] = (const uint32_t *)pb;
                    }
                    pos = pos_of[i];
                }
                int mtiles = 1;
                while (d * nB * mtiles < 296 && mtiles * MX_T < wo_max) mtiles *= 2;
                n.tiles = (pe >= 0) ? mtiles : 1;
                const int per_tile = (wo_max + n.tiles - 1) / n.tiles;
                const size_t sm = size_t(2) * (n.w[n.qc] + 1) * 8 + size_t(per_tile) * 4 + 16;
                if (sm + 2 * MX_T * 8 + 512 > 227 * 1024) return fail(SK_EOVERFLOW, "estimate: merged contraction too wide");
                SKB_CUDA(cudaFuncSetAttribute(k_node_merged_m, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                k_node_merged_m<<<dim3(d * nB, n.tiles), MX_T, sm, stream>>>(n, md, pos); count_launch();
            } else {
                if (pe < 0) {
                    // root: the outer leg is split over enough CTAs to fill the GPU, partials per
                    // tile in their own buffer (reduced below)
                    int qo = -1;
                    for (int q = 0; q < n.nl && qo < 0; ++q)
                        if (n.role[q] == RCHILD) qo = q;
                    const int wo_r = qo >= 0 ? n.w[qo] : 1;
                    int rt = 1;
                    while (blocks_xy * rt < 592 && rt * 256 < wo_r && rt < 64) rt *= 2;
                    if (rt > 1) {
                        void *pd;
                        if ((st = dalloc(pool, size_t(K) * d * nB * rt * 8, stream, &pd))) return st;
                        n.out = (uint64_t *)pd;
                        n.tiles = tiles = rt;
                        dense_root_part = (uint64_t *)pd;
                        dense_root_slots = nB * rt;
                    }
                }
                k_node_dense<<<dim3(blocks_xy, tiles), 256, 0, stream>>>(n, md); count_launch();
            }
            SKB_CUDA_CHECK("estimate launch 4");
        }
        if (exact) { k_root_reduce_x<<<d, 256, 0, stream>>>((const i128 *)part, (i128 *)acc, B * tiles_root); count_launch(); }
        else if (absb) { k_root_reduce_abs<<<d, 256, 0, stream>>>((const double *)part, (double *)acc, B * tiles_root); count_launch(); }
        else if (dense_root_part) {
            k_root_reduce<<<K * d, 256, 0, stream>>>(dense_root_part, acc, dense_root_slots, d, md); count_launch();
        } else { k_root_reduce<<<K * d, 256, 0, stream>>>((const uint64_t *)part, acc, B * tiles_root, d, md); count_launch(); }
        SKB_CUDA_CHECK("estimate launch 5");
    }
    return SK_OK;
}

// Evaluate a batch of sub-plans: all kernels enqueued, one device->host copy, one sync.
// The moduli come from the survivor bound (a sketch row built from N tuples has
// ||row||_1 <= N); the device-measured L1 norms verify it, else the plan is redone.
static bool is_two_way(const Plan &P) { return P.T.size() == 2 && P.T[0].kind == KV && P.T[1].kind == KV; }

// all two-way plans of a batch: one k_dot128 launch per kMaxDot plans, one copy, one sync.
// Plans with a flagged row are returned in `redo` (evaluated by the general engine).
static sk_status run_two_way(std::vector<Plan> &plans, const std::vector<size_t> &idx,
                             std::vector<std::vector<SBig>> &rows, std::vector<size_t> &redo, cudaStream_t stream) {
    if (idx.empty()) return SK_OK;
    int d = plans[idx[0]].d;
    for (size_t i : idx) d = std::max(d, plans[i].d);
    DevPool pool;
    void *dout;
    sk_status st;
    if ((st = dalloc(pool, idx.size() * d * 24, stream, &dout))) return st;
    uint64_t *out = (uint64_t *)dout;
    for (size_t b0 = 0; b0 < idx.size();) {
        // one launch per run of plans with equal d (grid = items x d)
        DotItems items;
        items.n = 0;
        items.d = plans[idx[b0]].d;
        size_t b1 = b0;
        while (b1 < idx.size() && items.n < kMaxDot && plans[idx[b1]].d == items.d) {
            const Plan &P = plans[idx[b1]];
            const sk_sketch *a = P.T[0].sk[0], *b = P.T[1].sk[0];
            items.it[items.n++] = {a->counters, b->counters, a->w[0], b->w[0], (uint32_t)P.width[0]};
            ++b1;
        }
        k_dot128<<<items.n * items.d, 512, 0, stream>>>(items, out + b0 * d * 3); count_launch();
        SKB_CUDA_CHECK("k_dot128 launch");
        b0 = b1;
    }
    std::vector<uint64_t> host(idx.size() * d * 3);
    SKB_CUDA(cudaMemcpyAsync(host.data(), out, host.size() * 8, cudaMemcpyDeviceToHost, stream));
    SKB_CUDA(cudaStreamSynchronize(stream));
    // items of one launch are laid out [item][d_launch][3] from the launch's base b0 * d * 3
    for (size_t b0 = 0; b0 < idx.size();) {
        const int dl = plans[idx[b0]].d;
        size_t b1 = b0;
        while (b1 < idx.size() && b1 - b0 < (size_t)kMaxDot && plans[idx[b1]].d == dl) ++b1;
        for (size_t j = b0; j < b1; ++j) {
            auto &rr = rows[idx[j]];
            rr.clear();
            const uint64_t *h = host.data() + b0 * d * 3 + (j - b0) * dl * 3;
            bool bad = false;
            for (int r = 0; r < dl; ++r) {
                rr.push_back(sbig_from_i128(h[3 * r], h[3 * r + 1]));
                bad |= h[3 * r + 2] != 0;
            }
            if (bad) { rr.clear(); redo.push_back(idx[j]); }
        }
        b0 = b1;
    }
    return SK_OK;
}

static sk_status run_batch(const sk_graph *g, std::vector<Plan> &plans, std::vector<std::vector<SBig>> &rows,
                           cudaStream_t stream, bool no_two_way = false, BatchShare *share = nullptr) {
    const size_t n = plans.size();
    rows.assign(n, {});
    if (!n) return SK_OK;
    // two-way sub-plans: exact int128 dot products; everything else: the CRT engine below
    {
        std::vector<size_t> tw;
        std::vector<Plan> rest;
        std::vector<size_t> rest_idx;
        for (size_t i = 0; i < n; ++i) {
            if (!no_two_way && is_two_way(plans[i]) && !getenv("COMPASS_EST_CRT_ONLY")) tw.push_back(i);
            else rest_idx.push_back(i);
        }
        if (!tw.empty()) {
            std::vector<size_t> redo;
            sk_status st = run_two_way(plans, tw, rows, redo, stream);
            if (st) return st;
            for (size_t i : redo) rest_idx.push_back(i);   // not provably exact in int128: CRT engine
            if (rest_idx.empty()) return SK_OK;
            for (size_t i : rest_idx) rest.push_back(std::move(plans[i]));
            std::vector<std::vector<SBig>> rrows;
            st = run_batch(g, rest, rrows, stream, /*no_two_way=*/true, share);
            for (size_t j = 0; j < rest_idx.size(); ++j) {
                plans[rest_idx[j]] = std::move(rest[j]);
                rows[rest_idx[j]] = std::move(rrows[j]);
            }
            return st;
        }
    }
    std::vector<Mods> mds(n);
    std::vector<std::vector<const sk_sketch *>> uniqs(n);
    std::vector<size_t> off_acc(n), off_l1(n);
    std::vector<char> exact(n, 0);
    std::vector<size_t> need_abs;
    std::vector<double> abs_bound(n, INFINITY);   // log2 of the absolute-value bound, when computed
    size_t words = 0;
    const bool crt_only = getenv("COMPASS_EST_CRT_ONLY") != nullptr;
    for (size_t i = 0; i < n; ++i) {
        Plan &P = plans[i];
        bool has_mat = false;
        for (auto &t : P.T) {
            has_mat |= t.kind == KM || t.kind == KT;
            for (auto *s : t.sk)
                if (std::find(uniqs[i].begin(), uniqs[i].end(), s) == uniqs[i].end()) uniqs[i].push_back(s);
        }
        const double logB = log_bound(P, [&](const sk_sketch *) { return 0.0; }) +
                            [&] { double v = 0; for (int t : P.tabs) v += log2(std::max<double>(1.0, (double)g->survivors[t])); return v; }();
        mds[i] = mods_for(logB, 1);
        // exact int128 contraction when the survivor bound fits (verified below with the
        // device-measured L1 norms) and the sub-plan has no matrix node
        exact[i] = !crt_only && !has_mat && logB <= 125.0;
        if (!crt_only && !has_mat && !exact[i]) need_abs.push_back(i);
        if (exact[i]) words = (words + 1) & ~size_t(1);   // int128 accumulators: 16-byte aligned
        off_acc[i] = words;
        words += size_t(exact[i] ? 2 : mds[i].K) * P.d;
        off_l1[i] = words;
        words += uniqs[i].size() * P.d;
    }
    // absolute-value bound pass (one batch, one sync) for matrix-free sub-plans whose survivor
    // bound exceeds int128: a bound A_r(1 + 2^-16) <= 2^125 on every row moves the plan to the
    // exact engine, else the moduli are sized from it
    if (!need_abs.empty()) {
        DevPool apool;
        void *dab;
        sk_status sa;
        const size_t aw = need_abs.size() * 64;
        if ((sa = dalloc(apool, aw * 8 + 8 * 64 * need_abs.size() * 64, stream, &dab))) return sa;
        SKB_CUDA(cudaMemsetAsync(dab, 0, aw * 8, stream));
        unsigned long long *l1s = (unsigned long long *)dab + aw;
        SKB_CUDA(cudaMemsetAsync(l1s, 0, 8 * 64 * need_abs.size() * 64, stream));
        for (size_t j = 0; j < need_abs.size(); ++j) {
            const size_t i = need_abs[j];
            if (plans[i].d > 64 || uniqs[i].size() > 64) continue;
            if ((sa = enqueue_plan(plans[i], mds[i], uniqs[i], apool, (uint64_t *)dab + j * 64, l1s + j * 64 * 64, stream, 2)))
                return sa;
        }
        std::vector<double> hb(aw);
        SKB_CUDA(cudaMemcpyAsync(hb.data(), dab, aw * 8, cudaMemcpyDeviceToHost, stream));
        SKB_CUDA(cudaStreamSynchronize(stream));
        size_t w2 = 0;
        for (size_t i = 0; i < n; ++i) {
            auto it = std::find(need_abs.begin(), need_abs.end(), i);
            if (it != need_abs.end() && plans[i].d <= 64 && uniqs[i].size() <= 64) {
                const size_t j = it - need_abs.begin();
                double mx = 0;
                for (int r = 0; r < plans[i].d; ++r) mx = std::max(mx, hb[j * 64 + r]);
                const double lb = log2(std::max(1.0, mx * (1.0 + 1.0 / 65536.0)));
                if (lb <= 125.0) exact[i] = 1;
                else mds[i] = mods_for(lb, 1);
                abs_bound[i] = lb;
            }
            if (exact[i]) w2 = (w2 + 1) & ~size_t(1);
            off_acc[i] = w2;
            w2 += size_t(exact[i] ? 2 : mds[i].K) * plans[i].d;
            off_l1[i] = w2;
            w2 += uniqs[i].size() * plans[i].d;
        }
        words = w2;
    }
    DevPool pool;
    void *dres;
    sk_status st;
    if ((st = dalloc(pool, words * 8, stream, &dres))) return st;
    SKB_CUDA(cudaMemsetAsync(dres, 0, words * 8, stream));
    uint64_t *res = (uint64_t *)dres;
    // matrix residues shared by every CRT plan of the batch (the first K_max primes; a plan
    // with K moduli uses the first K)
    Mods kmax_mods;
    kmax_mods.K = 0;
    for (size_t i = 0; i < n; ++i)
        if (!exact[i] && mds[i].K > kmax_mods.K) kmax_mods = mds[i];
    ResCache rescache;
    if (share) {
        rescache.shared = &share->by_K[kmax_mods.K];
        rescache.spool = &share->pool;
        rescache.stable = &share->stable;
    }
    // exact plans: 64-bit merged nodes where the survivor-based node bound is <= 2^61
    // (re-checked below with the measured L1 norms)
    std::vector<std::vector<char>> narrow(n);
    auto logF_of = [&](const Plan &P, auto l1of) {
        std::vector<double> f;
        for (auto &t : P.T) {
            double m = 0;
            for (auto *sk : t.sk) m = std::max(m, log2(std::max(1.0, l1of(sk))));
            f.push_back(m);
        }
        return f;
    };
    for (size_t i = 0; i < n; ++i) {
        if (!exact[i]) continue;
        const Plan &P = plans[i];
        std::vector<double> f;
        for (auto &t : P.T) f.push_back(log2(std::max<double>(1.0, (double)g->survivors[t.t])));
        std::vector<double> lb;
        node_logbounds(P, f, lb);
        narrow[i].assign(P.T.size(), 0);
        for (size_t j = 0; j < P.T.size(); ++j) narrow[i][j] = P.T[j].kind == KG && lb[j] <= 61.0;
    }
    // L1 norms once per distinct sketch of the batch (one k_l1 launch per 48 sketches), then
    // scattered into each plan's slots on the host after the copy
    std::vector<const sk_sketch *> guniq;
    std::map<const sk_sketch *, size_t> gidx;
    for (size_t i = 0; i < n; ++i)
        for (auto *sk : uniqs[i])
            if (!gidx.count(sk)) { gidx[sk] = guniq.size(); guniq.push_back(sk); }
    int dmax = 1;
    for (auto &P : plans) dmax = std::max(dmax, P.d);
    // norms already measured by an earlier batch of this planning call are reused (the
    // sketches cannot change while it runs); the rest are measured now
    std::vector<const sk_sketch *> l1todo;
    for (auto *sk : guniq)
        if (!(share && share->l1.count(sk))) l1todo.push_back(sk);
    void *dl1;
    if ((st = dalloc(pool, l1todo.size() * dmax * 8 + 8, stream, &dl1))) return st;
    SKB_CUDA(cudaMemsetAsync(dl1, 0, l1todo.size() * dmax * 8 + 8, stream));
    for (size_t b0 = 0; b0 < l1todo.size(); b0 += kMaxL1Items) {
        L1Items items;
        items.n = (int)std::min<size_t>(kMaxL1Items, l1todo.size() - b0);
        uint32_t maxcells = 1;
        for (int j = 0; j < items.n; ++j) {
            const sk_sketch *sk = l1todo[b0 + j];
            items.it[j] = {sk->counters, sk->d, (uint32_t)(sk->n_counters / sk->d)};
            maxcells = std::max(maxcells, items.it[j].cells);
        }
        const unsigned chunks = std::min<unsigned>(64, (maxcells + 8191) / 8192);
        k_l1<<<dim3(items.n, dmax, chunks), 256, 0, stream>>>(items, (unsigned long long *)dl1 + b0 * dmax, dmax);
        count_launch();
        SKB_CUDA_CHECK("estimate launch l1");
    }
    std::map<std::tuple<const void *, int, int>, const int64_t *> foldcache;
    std::map<std::pair<const void *, int>, std::array<void *, 4>> sortcache;
    std::map<std::vector<const void *>, std::array<const uint32_t *, 3>> rankcache;
    for (size_t i = 0; i < n; ++i)
        if ((st = enqueue_plan(plans[i], mds[i], uniqs[i], pool, res + off_acc[i], nullptr, stream, exact[i] ? 1 : 0,
                               &rescache, &kmax_mods, exact[i] ? &narrow[i] : nullptr, &foldcache, &sortcache, &rankcache)))
            return st;
    std::vector<uint64_t> host(words), hl1(guniq.size() * dmax), hnew(l1todo.size() * dmax);
    SKB_CUDA(cudaMemcpyAsync(host.data(), res, words * 8, cudaMemcpyDeviceToHost, stream));
    if (!hnew.empty()) SKB_CUDA(cudaMemcpyAsync(hnew.data(), dl1, hnew.size() * 8, cudaMemcpyDeviceToHost, stream));
    SKB_CUDA(cudaStreamSynchronize(stream));
    for (size_t j = 0; j < l1todo.size(); ++j) {
        std::copy(hnew.begin() + j * dmax, hnew.begin() + (j + 1) * dmax, hl1.begin() + gidx[l1todo[j]] * dmax);
        if (share) share->l1[l1todo[j]] = std::vector<uint64_t>(hnew.begin() + j * dmax, hnew.begin() + (j + 1) * dmax);
    }
    if (share)
        for (size_t j = 0; j < guniq.size(); ++j) {
            const auto &v = share->l1[guniq[j]];
            for (int r = 0; r < dmax && r < (int)v.size(); ++r) hl1[j * dmax + r] = v[r];
        }
    for (size_t i = 0; i < n; ++i)   // each plan's L1 slots, as enqueue_plan would have written them
        for (size_t u = 0; u < uniqs[i].size(); ++u)
            for (int r = 0; r < plans[i].d; ++r) host[off_l1[i] + u * plans[i].d + r] = hl1[gidx[uniqs[i][u]] * dmax + r];
    for (size_t i = 0; i < n; ++i) {
        const Plan &P = plans[i];
        const int d = P.d;
        auto l1of = [&](const sk_sketch *s) {
            const size_t u = std::find(uniqs[i].begin(), uniqs[i].end(), s) - uniqs[i].begin();
            uint64_t mx = 0;
            for (int r = 0; r < d; ++r) mx = std::max<uint64_t>(mx, host[off_l1[i] + u * d + r]);
            // saturated (>= 2^64): the worst case for int64 counters, 2^63 per cell
            if (mx == ~0ULL) return ldexp((double)(s->n_counters / s->d), 63);
            return (double)mx;
        };
        const double logB = std::min(log_bound(P, l1of), abs_bound[i]);
        bool narrow_ok = true;
        if (exact[i]) {   // 64-bit nodes must also hold under the measured norms
            std::vector<double> lb;
            node_logbounds(P, logF_of(P, l1of), lb);
            for (size_t j = 0; j < P.T.size(); ++j)
                if (narrow[i][j] && lb[j] > 61.0) narrow_ok = false;   // re-run on the CRT engine below
        }
        if (exact[i] && narrow_ok && logB <= 125.0) {
            for (int r = 0; r < d; ++r) rows[i].push_back(sbig_from_i128(host[off_acc[i] + 2 * r], host[off_acc[i] + 2 * r + 1]));
            continue;
        }
        if (exact[i] || logB + 3.0 > mods_capacity(mds[i])) {
            // the survivor bound did not hold for these sketches: redo with the measured bound
            Mods md = mods_for(logB, 1);
            if (mods_capacity(md) < logB + 3.0)
                return fail(SK_EOVERFLOW, "estimate: bound 2^%.1f exceeds the exact range", logB);
            DevPool pool2;
            void *d2;
            const size_t w2 = size_t(md.K) * d + uniqs[i].size() * d;
            if ((st = dalloc(pool2, w2 * 8, stream, &d2))) return st;
            SKB_CUDA(cudaMemsetAsync(d2, 0, w2 * 8, stream));
            if ((st = enqueue_plan(P, md, uniqs[i], pool2, (uint64_t *)d2, (unsigned long long *)d2 + size_t(md.K) * d, stream)))
                return st;
            std::vector<uint64_t> h2(w2);
            SKB_CUDA(cudaMemcpyAsync(h2.data(), d2, w2 * 8, cudaMemcpyDeviceToHost, stream));
            SKB_CUDA(cudaStreamSynchronize(stream));
            for (int r = 0; r < d; ++r) {
                uint64_t rr[kMaxMod];
                for (int k = 0; k < md.K; ++k) rr[k] = h2[size_t(k) * d + r];
                rows[i].push_back(crt_signed(rr, md));
            }
            continue;
        }
        for (int r = 0; r < d; ++r) {
            uint64_t rr[kMaxMod];
            for (int k = 0; k < mds[i].K; ++k) rr[k] = host[off_acc[i] + size_t(k) * d + r];
            rows[i].push_back(crt_signed(rr, mds[i]));
        }
    }
    return SK_OK;
}

}  // namespace

namespace skb {

// Batched evaluation: masks[i] -> est[i] (median, fp64), optional per-row values.
sk_status estimate_batch(const sk_graph *g, const uint64_t *masks, uint32_t n, double *est,
                         std::vector<std::vector<SBig>> *rows_out, cudaStream_t stream, BatchShare *share = nullptr) {
    if (!g) return fail(SK_EINVAL, "estimate: NULL graph");
    std::vector<Plan> plans;
    std::vector<uint32_t> which;
    for (uint32_t i = 0; i < n; ++i) {
        const uint64_t mask = masks[i];
        const int pc = __builtin_popcountll(mask);
        if (pc == 0) return fail(SK_EINVAL, "estimate: empty vertex mask");
        if (pc == 1) {
            const int t = __builtin_ctzll(mask);
            if ((uint32_t)t >= g->n_tables || !g->survivors) return fail(SK_EINVAL, "estimate: bad singleton");
            if (est) est[i] = (double)g->survivors[t];
            continue;
        }
        if (!g->survivors) return fail(SK_EINVAL, "estimate: graph survivors missing");
        Plan P;
        sk_status st = build_plan(g, mask, P);
        if (st) return st;
        plans.push_back(std::move(P));
        which.push_back(i);
    }
    if (rows_out) rows_out->assign(n, {});
    if (plans.empty()) return SK_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    SKB_CUDA(cudaSetDevice(plans[0].device));
    std::vector<std::vector<SBig>> rows;
    sk_status st = run_batch(g, plans, rows, stream, false, share);
    cudaSetDevice(prev);
    if (st) return st;
    for (size_t j = 0; j < plans.size(); ++j) {
        const uint32_t i = which[j];
        std::vector<int> idx(rows[j].size());
        for (size_t r = 0; r < idx.size(); ++r) idx[r] = (int)r;
        std::sort(idx.begin(), idx.end(), [&](int x, int y) { return SBig::cmp(rows[j][x], rows[j][y]) < 0; });
        if (est) est[i] = rows[j][idx[(rows[j].size() - 1) / 2]].to_double();
        if (rows_out) (*rows_out)[i] = std::move(rows[j]);
    }
    return SK_OK;
}

sk_status estimate_mask(const sk_graph *g, uint64_t mask, double *est, double *row_est,
                        std::vector<std::string> *rows_exact, cudaStream_t stream) {
    std::vector<std::vector<SBig>> rows;
    double e = 0;
    sk_status st = estimate_batch(g, &mask, 1, &e, &rows, stream);
    if (st) return st;
    if (est) *est = e;
    if (row_est) for (size_t r = 0; r < rows[0].size(); ++r) row_est[r] = rows[0][r].to_double();
    if (rows_exact) { rows_exact->clear(); for (auto &v : rows[0]) rows_exact->push_back(v.to_dec()); }
    return SK_OK;
}

}  // namespace skb

extern "C" sk_status estimate_join(const sk_graph *g, uint64_t vertex_mask, double *est, double *row_est, void *stream) {
    return estimate_mask(g, vertex_mask, est, row_est, nullptr, (cudaStream_t)stream);
}

extern "C" sk_status estimate_join_exact(const sk_graph *g, uint64_t vertex_mask, char *buf, uint32_t stride, void *stream) {
    if (!buf || stride < 2) return fail(SK_EINVAL, "estimate_join_exact: bad buffer");
    std::vector<std::string> rows;
    double est;
    sk_status st = estimate_mask(g, vertex_mask, &est, nullptr, &rows, (cudaStream_t)stream);
    if (st) return st;
    if (__builtin_popcountll(vertex_mask) == 1) {
        snprintf(buf, stride, "%lld", (long long)est);
        return SK_OK;
    }
    for (size_t r = 0; r < rows.size(); ++r) {
        if (rows[r].size() + 1 > stride) return fail(SK_EINVAL, "estimate_join_exact: stride too small");
        memcpy(buf + r * stride, rows[r].c_str(), rows[r].size() + 1);
    }
    return SK_OK;
}

extern "C" sk_status estimate_subplans(const sk_graph *g, const uint64_t *masks, uint32_t n, double *est, void *stream) {
    if (n && (!masks || !est)) return fail(SK_EINVAL, "estimate_subplans: NULL array");
    return estimate_batch(g, masks, n, est, nullptr, (cudaStream_t)stream);
}

namespace skb {

// Estimate cache of one planning call: card(S) = survivors for |S| = 1,
// max(Est(S), 0) otherwise; all connected sub-plans are estimated in one batch up front when
// there are at most 512 of them, else on demand.
struct CardCache {
    const sk_graph *g;
    cudaStream_t stream;
    std::map<uint64_t, double> cache;
    sk_status err = SK_OK;
    uint64_t calls = 0;
    BatchShare share;   // matrix residues shared by the batches of this planning call
    CardCache(const sk_graph *g_, cudaStream_t s) : g(g_), stream(s), share(g_) {}
    sk_status prefetch() {
        const uint32_t n = g->n_tables;
        if (n > 16) return SK_OK;
        std::vector<uint64_t> adj(n, 0);
        for (uint32_t e = 0; e < g->n_edges; ++e) {
            if (g->edge_u[e] >= n || g->edge_v[e] >= n) return fail(SK_EINVAL, "planner: bad edge");
            adj[g->edge_u[e]] |= 1ULL << g->edge_v[e];
            adj[g->edge_v[e]] |= 1ULL << g->edge_u[e];
        }
        std::vector<uint64_t> masks;
        for (uint64_t m = 1; m < (1ULL << n) && masks.size() <= 512; ++m) {
            if (__builtin_popcountll(m) < 2) continue;
            uint64_t seen = m & (~m + 1), frontier = seen;
            while (frontier) {
                uint64_t nxt = 0;
                for (uint64_t f = frontier; f; f &= f - 1) nxt |= adj[__builtin_ctzll(f)];
                nxt &= m & ~seen;
                seen |= nxt;
                frontier = nxt;
            }
            if (seen == m) masks.push_back(m);
        }
        if (masks.size() > 512) return SK_OK;
        std::vector<double> est(masks.size());
        sk_status st = estimate_batch(g, masks.data(), (uint32_t)masks.size(), est.data(), nullptr, stream, &share);
        if (st) return st;
        for (size_t i = 0; i < masks.size(); ++i) cache[masks[i]] = std::max(est[i], 0.0);
        return SK_OK;
    }
    // one batch for the given sub-plans that are not cached yet (greedy: one batch per level,
    // only the sub-plans the enumeration reads)
    sk_status prefetch_masks(const std::vector<uint64_t> &want) {
        std::vector<uint64_t> masks;
        for (uint64_t m : want)
            if (__builtin_popcountll(m) >= 2 && !cache.count(m) &&
                std::find(masks.begin(), masks.end(), m) == masks.end())
                masks.push_back(m);
        if (masks.empty()) return SK_OK;
        std::vector<double> est(masks.size());
        sk_status st = estimate_batch(g, masks.data(), (uint32_t)masks.size(), est.data(), nullptr, stream, &share);
        if (st) return st;
        for (size_t i = 0; i < masks.size(); ++i) cache[masks[i]] = std::max(est[i], 0.0);
        return SK_OK;
    }
    double card(uint64_t m) {
        ++calls;
        auto it = cache.find(m);
        if (it != cache.end()) return it->second;
        double c;
        if (__builtin_popcountll(m) == 1) {
            c = (double)g->survivors[__builtin_ctzll(m)];
        } else {
            double e = 0;
            sk_status st = estimate_mask(g, m, &e, nullptr, nullptr, stream);
            if (st && !err) err = st;
            c = std::max(e, 0.0);
        }
        cache[m] = c;
        return c;
    }
};

// PAPER.md:662 greedy: cheapest two-vertex sub-plan, source = its endpoint with
// fewer survivors, then repeatedly the cheapest neighbour extension.
static sk_status greedy_order(CardCache &cc, std::vector<uint32_t> &C, std::vector<double> &pre) {
    const sk_graph *g = cc.g;
    const uint32_t n = g->n_tables;
    C.clear();
    pre.clear();
    if (n == 1) {
        C.push_back(0);
        pre.push_back(cc.card(1ULL));
        return cc.err;
    }
    int bu = -1, bv = -1;
    double bc = 0;
    {
        std::vector<uint64_t> lvl;
        for (uint32_t e = 0; e < g->n_edges; ++e) lvl.push_back((1ULL << g->edge_u[e]) | (1ULL << g->edge_v[e]));
        sk_status st = cc.prefetch_masks(lvl);
        if (st) return st;
    }
    for (uint32_t e = 0; e < g->n_edges; ++e) {
        int u = (int)std::min(g->edge_u[e], g->edge_v[e]), v = (int)std::max(g->edge_u[e], g->edge_v[e]);
        const double c = cc.card((1ULL << u) | (1ULL << v));
        if (cc.err) return cc.err;
        if (bu < 0 || c < bc || (c == bc && (u < bu || (u == bu && v < bv)))) { bu = u; bv = v; bc = c; }
    }
    if (bu < 0) return fail(SK_EINVAL, "planner: graph has no edges");
    const int src = (g->survivors[bv] < g->survivors[bu]) ? bv : bu;
    C.push_back((uint32_t)src);
    uint64_t m = 1ULL << src;
    pre.push_back(cc.card(m));
    while (C.size() < n) {
        int best = -1;
        double bcard = 0;
        {
            std::vector<uint64_t> lvl;   // every extension of C by one neighbour, one batch
            for (uint32_t e = 0; e < g->n_edges; ++e) {
                const uint32_t u = g->edge_u[e], v = g->edge_v[e];
                if (((m >> u) & 1ULL) && !((m >> v) & 1ULL)) lvl.push_back(m | (1ULL << v));
                if (((m >> v) & 1ULL) && !((m >> u) & 1ULL)) lvl.push_back(m | (1ULL << u));
            }
            sk_status st = cc.prefetch_masks(lvl);
            if (st) return st;
        }
        for (uint32_t e = 0; e < g->n_edges; ++e) {
            const uint32_t u = g->edge_u[e], v = g->edge_v[e];
            int cand = -1;
            if (((m >> u) & 1ULL) && !((m >> v) & 1ULL)) cand = (int)v;
            if (((m >> v) & 1ULL) && !((m >> u) & 1ULL)) cand = (int)u;
            if (cand < 0) continue;
            const double c = cc.card(m | (1ULL << cand));
            if (cc.err) return cc.err;
            if (best < 0 || c < bcard || (c == bcard && cand < best)) { best = cand; bcard = c; }
        }
        if (best < 0) return fail(SK_EINVAL, "planner: join graph is not connected");
        C.push_back((uint32_t)best);
        m |= 1ULL << best;
        pre.push_back(bcard);
    }
    return cc.err;
}

static sk_status check_graph(const sk_graph *g) {
    if (!g) return fail(SK_EINVAL, "planner: NULL graph");
    if (g->n_tables == 0 || g->n_tables > 64) return fail(SK_EINVAL, "planner: n_tables must be in [1,64]");
    if (!g->survivors) return fail(SK_EINVAL, "planner: graph survivors missing");
    for (uint32_t e = 0; e < g->n_edges; ++e)
        if (g->edge_u[e] >= g->n_tables || g->edge_v[e] >= g->n_tables || g->edge_u[e] == g->edge_v[e])
            return fail(SK_EINVAL, "planner: bad edge %u", e);
    return SK_OK;
}

// Algorithm 1: DFS Traversal with early pruning and a per-source plan limit
struct Enumerator {
    CardCache &cc;
    const sk_graph *g;
    uint32_t n;
    std::vector<uint64_t> adj;
    uint64_t max_plans;      // 0 = unbounded
    bool prune;
    double min_cost = INFINITY;
    std::vector<uint32_t> opt_path, C;
    uint64_t p = 0;          // plans completed from the current source
    bool abort_source = false;
    sk_enum_stats st{};
    Enumerator(CardCache &c, uint64_t mp, bool pr) : cc(c), g(c.g), n(c.g->n_tables), adj(n, 0), max_plans(mp), prune(pr) {
        for (uint32_t e = 0; e < g->n_edges; ++e) {
            adj[g->edge_u[e]] |= 1ULL << g->edge_v[e];
            adj[g->edge_v[e]] |= 1ULL << g->edge_u[e];
        }
    }
    void dfs(uint64_t m, double cost) {
        if (abort_source || cc.err) return;
        const double curr = cc.card(m);                       // line 14
        cost += curr;                                         // line 15
        if (prune && cost > min_cost) { ++st.prunes; return; }   // line 17
        if (C.size() == n) {                                  // lines 19-26
            if (cost < min_cost) { min_cost = cost; opt_path = C; }
            ++st.plans_completed;
            ++p;
            if (max_plans && p == max_plans) abort_source = true;
            return;
        }
        // lines 29-35: neighbours of C, in increasing card(C + v), ties by index
        uint64_t L = 0;
        for (uint64_t f = m; f; f &= f - 1) L |= adj[__builtin_ctzll(f)];
        L &= ~m;
        std::vector<std::pair<double, uint32_t>> ev;
        for (uint64_t f = L; f; f &= f - 1) {
            const uint32_t v = (uint32_t)__builtin_ctzll(f);
            ev.push_back({cc.card(m | (1ULL << v)), v});
        }
        std::sort(ev.begin(), ev.end());
        for (auto &e : ev) {
            if (abort_source || cc.err) return;
            C.push_back(e.second);
            dfs(m | (1ULL << e.second), cost);
            C.pop_back();
        }
    }
};

}  // namespace skb

extern "C" sk_status plan_greedy(const sk_graph *g, uint32_t *order, double *prefix_card, double *cost, void *stream) {
    if (!g || !order) return fail(SK_EINVAL, "plan_greedy: NULL argument");
    sk_status st = check_graph(g);
    if (st) return st;
    CardCache cc(g, (cudaStream_t)stream);   // greedy batches its reads level by level
    std::vector<uint32_t> C;
    std::vector<double> pre;
    if ((st = greedy_order(cc, C, pre))) return st;
    double total = 0;
    for (size_t i = 0; i < C.size(); ++i) {
        order[i] = C[i];
        if (prefix_card) prefix_card[i] = pre[i];
        total += pre[i];
    }
    if (cost) *cost = total;
    return SK_OK;
}

extern "C" sk_status plan_enumerate(const sk_graph *g, const sk_enum_config *cfg, uint32_t *order, double *prefix_card,
                                    double *cost, sk_enum_stats *stats, void *stream) {
    if (!g || !cfg || !order) return fail(SK_EINVAL, "plan_enumerate: NULL argument");
    sk_status st = check_graph(g);
    if (st) return st;
    if (cfg->mode > SK_ENUM_EXHAUSTIVE) return fail(SK_EINVAL, "plan_enumerate: unknown mode %u", cfg->mode);
    if (cfg->mode == SK_ENUM_LIMIT && cfg->max_plans == 0) return fail(SK_EINVAL, "plan_enumerate: max_plans must be >= 1");
    if (!(cfg->alpha >= 0) || !(cfg->beta >= 0)) return fail(SK_EINVAL, "plan_enumerate: alpha, beta must be >= 0");
    CardCache cc(g, (cudaStream_t)stream);
    if ((st = cc.prefetch())) return st;
    const uint32_t n = g->n_tables;
    std::vector<uint32_t> best;
    double best_cost = 0;
    sk_enum_stats es{};
    if (cfg->mode == SK_ENUM_GREEDY) {
        std::vector<double> pre;
        if ((st = greedy_order(cc, best, pre))) return st;
        for (double c : pre) best_cost += c;
        es.plans_completed = 1;
    } else {
        // line 7: sources in increasing f(v), ties by index
        std::vector<uint32_t> deg(n, 0);
        for (uint32_t e = 0; e < g->n_edges; ++e) { ++deg[g->edge_u[e]]; ++deg[g->edge_v[e]]; }
        double maxc = 0, maxd = 0;
        for (uint32_t v = 0; v < n; ++v) { maxc = std::max(maxc, (double)g->survivors[v]); maxd = std::max(maxd, (double)deg[v]); }
        std::vector<std::pair<double, uint32_t>> S;
        for (uint32_t v = 0; v < n; ++v) {
            const double f = (maxc > 0 ? cfg->alpha * (double)g->survivors[v] / maxc : 0.0) +
                             (maxd > 0 ? cfg->beta * (double)deg[v] / maxd : 0.0);
            S.push_back({f, v});
        }
        std::sort(S.begin(), S.end());
        const uint64_t mp = cfg->mode == SK_ENUM_FULL_GREEDY ? 1 : cfg->mode == SK_ENUM_LIMIT ? cfg->max_plans : 0;
        Enumerator en(cc, mp, !cfg->no_prune);
        for (auto &sv : S) {                                   // lines 8-11
            en.p = 0;
            en.abort_source = false;
            en.C.assign(1, sv.second);
            en.dfs(1ULL << sv.second, 0.0);
            if (cc.err) return cc.err;
        }
        if (en.opt_path.size() != n) return fail(SK_EINVAL, "plan_enumerate: join graph is not connected");
        best = en.opt_path;
        best_cost = en.min_cost;
        es = en.st;
    }
    if (cc.err) return cc.err;
    es.estimator_calls = cc.calls;
    es.distinct_estimates = cc.cache.size();
    uint64_t m = 0;
    for (size_t i = 0; i < best.size(); ++i) {
        order[i] = best[i];
        m |= 1ULL << best[i];
        if (prefix_card) prefix_card[i] = cc.card(m);
    }
    if (cost) *cost = best_cost;
    if (stats) *stats = es;
    return cc.err;
}

// Exact count of a connected sub-plan whose kept edges form a tree (frequency-vector message
// passing, one prime per blockIdx.y, CRT).  extra[t]: additional point predicates (column,
// value) on table t (cycle conditioning).
static sk_status exact_tree(const sk_join_data *jd, uint64_t mask, const std::vector<uint32_t> &ed,
                            const std::vector<std::vector<std::pair<uint32_t, int64_t>>> &extra, cudaStream_t stream,
                            SBig *out) {
    const uint32_t T = jd->n_tables;
    const int nC = __builtin_popcountll(mask);
    const int root = __builtin_ctzll(mask);
    // DFS from the root: parent edge per table, post-order
    std::vector<int> pe(T, -2), order;
    {
        std::vector<int> st{root}, pre;
        pe[root] = -1;
        while (!st.empty()) {
            const int x = st.back();
            st.pop_back();
            pre.push_back(x);
            for (uint32_t e : ed) {
                const int u = (int)jd->edge_u[e], v = (int)jd->edge_v[e];
                const int y = u == x ? v : (v == x ? u : -1);
                if (y < 0 || pe[y] != -2) continue;
                pe[y] = (int)e;
                st.push_back(y);
            }
        }
        if ((int)pre.size() != nC) return fail(SK_EINVAL, "exact_join_size: sub-plan is not connected");
        order.assign(pre.rbegin(), pre.rend());
    }
    double logB = 1;
    for (int t : order) logB += log2(std::max<double>(1.0, (double)jd->tables[t].n_rows));
    const Mods md = mods_for(logB, 1);
    int prev = 0;
    cudaGetDevice(&prev);
    DevPool pool;
    sk_status st;
    void *derr, *dacc;
    if ((st = dalloc(pool, 16, stream, &derr))) return st;
    if ((st = dalloc(pool, size_t(md.K) * 8, stream, &dacc))) return st;
    SKB_CUDA(cudaMemsetAsync(derr, 0, 16, stream));
    SKB_CUDA(cudaMemsetAsync(dacc, 0, size_t(md.K) * 8, stream));
    std::vector<uint64_t *> msg(jd->n_edges, nullptr);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, prev);
    for (int t : order) {
        const sk_table_data &td = jd->tables[t];
        XNode n;
        memset(&n, 0, sizeof(n));
        if (td.n_preds + extra[t].size() > (size_t)kXPreds)
            return fail(SK_EOVERFLOW, "exact_join_size: table %d has too many predicates for cycle conditioning", t);
        n.n_rows = td.n_rows;
        for (uint32_t c = 0; c < td.n_cols; ++c) {
            if (!td.cols[c].data && td.n_rows) return fail(SK_EINVAL, "exact_join_size: table %d column %u is NULL", t, c);
            n.col[c] = td.cols[c].data;
            if (td.cols[c].dtype == SK_INT64) n.col64 |= 1u << c;
            else if (td.cols[c].dtype != SK_INT32) return fail(SK_EINVAL, "exact_join_size: bad dtype");
        }
        n.n_preds = td.n_preds;
        for (uint32_t q = 0; q < td.n_preds; ++q) {
            const sk_pred &pr = td.preds[q];
            n.pred[q] = XPred{pr.col, pr.kind, pr.lo, pr.hi, nullptr, 0};
            if (pr.kind == SK_PRED_SUBSET) {
                if (pr.set_size && !pr.set) return fail(SK_EINVAL, "exact_join_size: NULL subset");
                std::vector<int64_t> sv(pr.set, pr.set + pr.set_size);
                std::sort(sv.begin(), sv.end());
                sv.erase(std::unique(sv.begin(), sv.end()), sv.end());
                n.pred[q].n = (uint32_t)sv.size();
                if (!sv.empty()) {
                    void *ds;
                    if ((st = dalloc(pool, sv.size() * 8, stream, &ds))) return st;
                    SKB_CUDA(cudaMemcpyAsync(ds, sv.data(), sv.size() * 8, cudaMemcpyHostToDevice, stream));
                    n.pred[q].set = (const int64_t *)ds;
                }
            }
        }
        for (const auto &xp : extra[t]) n.pred[n.n_preds++] = XPred{xp.first, SK_PRED_POINT, xp.second, xp.second, nullptr, 0};
        for (uint32_t e : ed) {
            if ((int)e == pe[t]) continue;
            const bool at_u = (int)jd->edge_u[e] == t, at_v = (int)jd->edge_v[e] == t;
            if (!at_u && !at_v) continue;
            if (n.n_child == (uint32_t)kXChild) return fail(SK_EOVERFLOW, "exact_join_size: table %d has > 4 sub-plan edges", t);
            n.ch[n.n_child++] = XChild{msg[e], at_u ? jd->col_u[e] : jd->col_v[e], jd->key_lo[e], jd->key_domain[e]};
        }
        if (pe[t] >= 0) {
            const uint32_t e = (uint32_t)pe[t];
            void *mb;
            if ((st = dalloc(pool, size_t(md.K) * jd->key_domain[e] * 8, stream, &mb))) return st;
            SKB_CUDA(cudaMemsetAsync(mb, 0, size_t(md.K) * jd->key_domain[e] * 8, stream));
            msg[e] = (uint64_t *)mb;
            n.has_parent = 1;
            n.pcol = (int)jd->edge_u[e] == t ? jd->col_u[e] : jd->col_v[e];
            n.plo = jd->key_lo[e];
            n.pdom = jd->key_domain[e];
            n.out = msg[e];
        } else {
            n.out = (uint64_t *)dacc;
        }
        const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(sms) * 4, (td.n_rows + 255) / 256));
        k_exact_node<<<dim3(gx, md.K), 256, 0, stream>>>(n, md, (unsigned int *)derr); count_launch();
        SKB_CUDA_CHECK("k_exact_node launch");
        if (pe[t] >= 0) {
            const uint64_t dom = jd->key_domain[pe[t]];
            k_mod_reduce<<<dim3((unsigned)std::min<uint64_t>(uint64_t(sms) * 4, (dom + 255) / 256), md.K), 256, 0, stream>>>(
                msg[pe[t]], dom, md);
            count_launch();
        }
    }
    uint64_t herr[2] = {0, 0};
    std::vector<uint64_t> hacc(md.K);
    SKB_CUDA(cudaMemcpyAsync(herr, derr, 16, cudaMemcpyDeviceToHost, stream));
    SKB_CUDA(cudaMemcpyAsync(hacc.data(), dacc, size_t(md.K) * 8, cudaMemcpyDeviceToHost, stream));
    SKB_CUDA(cudaStreamSynchronize(stream));
    if (herr[0] & 0xffffffffu) return fail(SK_EINVAL, "exact_join_size: a join key lies outside its edge's key domain");
    for (int k = 0; k < md.K; ++k) hacc[k] %= md.m[k];
    *out = crt_signed(hacc.data(), md);
    if (out->neg && !out->mag.zero()) return fail(SK_ECUDA, "exact_join_size: negative count (internal error)");
    return SK_OK;
}

// union-find over (table, column) nodes: equality of join keys is transitive, so an induced
// edge whose two columns are already equal through the other kept edges is implied (e.g. the
// C3 triangle T.id = MK.mid = CI.mid) and dropped without changing the count
static uint32_t uf_find(std::vector<uint32_t> &p, uint32_t x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
}

// Exact count of any connected sub-plan: implied edges dropped; a remaining cycle is
// conditioned on one of its edges (u.cu = v.cv = k for every k of the edge's key domain,
// each an acyclic count with two more point predicates), recursively.
static sk_status exact_any(const sk_join_data *jd, uint64_t mask, std::vector<uint32_t> ed,
                           std::vector<std::vector<std::pair<uint32_t, int64_t>>> extra, cudaStream_t stream,
                           uint64_t &budget, SBig *out) {
    const uint32_t T = jd->n_tables;
    const int nC = __builtin_popcountll(mask);
    std::vector<uint32_t> par(T * (uint32_t)kXCols);
    for (uint32_t i = 0; i < par.size(); ++i) par[i] = i;
    std::vector<uint32_t> kept;
    std::vector<uint32_t> tpar(T);   // table-level union-find: the first edge closing a table cycle
    for (uint32_t i = 0; i < T; ++i) tpar[i] = i;
    int cyc = -1;
    for (uint32_t e : ed) {
        const uint32_t a = uf_find(par, jd->edge_u[e] * kXCols + jd->col_u[e]);
        const uint32_t b = uf_find(par, jd->edge_v[e] * kXCols + jd->col_v[e]);
        if (a == b) continue;   // implied by transitivity
        par[a] = b;
        kept.push_back(e);
        const uint32_t ta = uf_find(tpar, jd->edge_u[e]), tb = uf_find(tpar, jd->edge_v[e]);
        if (ta == tb) { if (cyc < 0) cyc = (int)e; }
        else tpar[ta] = tb;
    }
    if ((int)kept.size() < nC - 1) return fail(SK_EINVAL, "exact_join_size: sub-plan is not connected");
    if (cyc < 0) return exact_tree(jd, mask, kept, extra, stream, out);
    // a genuine cycle: condition the edge that closed it on every key of its domain
    const uint32_t e = (uint32_t)cyc;
    const uint64_t dom = jd->key_domain[e];
    if (dom > budget) return fail(SK_EOVERFLOW, "exact_join_size: cycle conditioning over %llu keys exceeds the limit",
                                  (unsigned long long)dom);
    budget -= dom;
    std::vector<uint32_t> rest;
    for (uint32_t f : kept) if (f != e) rest.push_back(f);
    out->neg = false;
    out->mag = UBig();
    for (uint64_t i = 0; i < dom; ++i) {
        const int64_t k = jd->key_lo[e] + (int64_t)i;
        auto ex = extra;
        ex[jd->edge_u[e]].push_back({jd->col_u[e], k});
        ex[jd->edge_v[e]].push_back({jd->col_v[e], k});
        SBig part;
        sk_status st = exact_any(jd, mask, rest, ex, stream, budget, &part);
        if (st) return st;
        out->mag = UBig::add(out->mag, part.mag);
    }
    return SK_OK;
}

extern "C" sk_status exact_join_size(const sk_join_data *jd, uint64_t mask, char *dec, uint32_t dec_len, double *approx,
                                     void *stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (!jd || !jd->tables) return fail(SK_EINVAL, "exact_join_size: NULL argument");
    if (dec && dec_len < 2) return fail(SK_EINVAL, "exact_join_size: dec_len must be >= 2");
    const uint32_t T = jd->n_tables;
    if (T == 0 || T > 64) return fail(SK_EINVAL, "exact_join_size: n_tables must be in [1,64]");
    if (mask == 0 || (T < 64 && (mask >> T))) return fail(SK_EINVAL, "exact_join_size: bad vertex mask");
    for (uint32_t t = 0; t < T; ++t) {
        const sk_table_data &td = jd->tables[t];
        if (td.n_cols > (uint32_t)kXCols || td.n_preds > (uint32_t)kXPreds)
            return fail(SK_EINVAL, "exact_join_size: table %u has too many columns/predicates", t);
        if ((td.n_cols && !td.cols) || (td.n_preds && !td.preds)) return fail(SK_EINVAL, "exact_join_size: NULL array");
        for (uint32_t q = 0; q < td.n_preds; ++q)
            if (td.preds[q].col >= td.n_cols || td.preds[q].kind > SK_PRED_SUBSET)
                return fail(SK_EINVAL, "exact_join_size: table %u predicate %u invalid", t, q);
    }
    // induced edges; acyclic and connected (|E_C| = |C| - 1)
    std::vector<uint32_t> ed;
    for (uint32_t e = 0; e < jd->n_edges; ++e) {
        const uint32_t u = jd->edge_u[e], v = jd->edge_v[e];
        if (u >= T || v >= T || u == v) return fail(SK_EINVAL, "exact_join_size: bad edge %u", e);
        if (jd->col_u[e] >= jd->tables[u].n_cols || jd->col_v[e] >= jd->tables[v].n_cols)
            return fail(SK_EINVAL, "exact_join_size: edge %u column out of range", e);
        if (jd->key_domain[e] == 0 || jd->key_domain[e] > (1ULL << 31))
            return fail(SK_EINVAL, "exact_join_size: edge %u key domain must be in [1, 2^31]", e);
        if (((mask >> u) & 1ULL) && ((mask >> v) & 1ULL)) ed.push_back(e);
    }
    const int nC = __builtin_popcountll(mask);
    if ((int)ed.size() < nC - 1) return fail(SK_EINVAL, "exact_join_size: sub-plan is not connected");
    int prev = 0;
    cudaGetDevice(&prev);
    std::vector<std::vector<std::pair<uint32_t, int64_t>>> extra(T);
    uint64_t budget = 1ULL << 16;   // total conditioned keys (cycles of small key domains only)
    SBig v;
    sk_status st = exact_any(jd, mask, ed, extra, stream, budget, &v);
    if (st) return st;
    if (dec) {
        const std::string sd = v.to_dec();
        if (sd.size() + 1 > dec_len) return fail(SK_EINVAL, "exact_join_size: dec_len too small");
        memcpy(dec, sd.c_str(), sd.size() + 1);
    }
    if (approx) *approx = v.to_double();
    return SK_OK;
}
