// hash.cuh — device arithmetic mod the Mersenne prime p = 2^61 - 1 for the
// Fast-AGMS hash family (the paper fixes no family,
// PAPER.md:152; SPEC.md:69-71 chooses these polynomials).
#pragma once
#include <stdint.h>

#define SKH_P 0x1FFFFFFFFFFFFFFFULL

// H1: sign-extended key reinterpreted as uint64, reduced mod p.
__device__ __forceinline__ uint64_t canon61(int64_t key) {
    const uint64_t u = (uint64_t)key;
    const uint64_t x = (u & SKH_P) + (u >> 61);
    return x >= SKH_P ? x - SKH_P : x;
}

// v < 2^62  ->  v mod p
__device__ __forceinline__ uint64_t red61(uint64_t v) {
    v = (v & SKH_P) + (v >> 61);
    return v >= SKH_P ? v - SKH_P : v;
}

// a, b < p  ->  a*b mod p   (2^64 = 8 * 2^61 = 8 mod p)
__device__ __forceinline__ uint64_t mulmod61(uint64_t a, uint64_t b) {
    const uint64_t lo = a * b;
    const uint64_t hi = __umul64hi(a, b);
    const uint64_t r = (lo & SKH_P) + (lo >> 61) + (hi << 3);
    return red61(r);
}

// Lazily reduced v*x mod p for a key x < 2^32 (every int32 key >= 0 and most dense key
// domains): two 32x32->64 products instead of a 64x64->128 one.  v < 2^64; the result is
// congruent to v*x mod p and < 2^62 + 2^35 + 8 (not fully reduced).
//   v*x = p1 + p2*2^32, p1 = vlo*x, p2 = vhi*x;  p1 = (p1 & p) + (p1 >> 61) (mod p);
//   p2*2^32 = (p2 >> 29)*2^61 + (p2 & (2^29-1))*2^32 == (p2 >> 29) + ((p2 & (2^29-1)) << 32).
__device__ __forceinline__ uint64_t mulmod61_x32(uint64_t v, uint32_t x) {
    const uint64_t p1 = (uint64_t)(uint32_t)v * x;
    const uint64_t p2 = (uint64_t)(uint32_t)(v >> 32) * x;
    return (p1 & SKH_P) + (p1 >> 61) + (p2 >> 29) + ((p2 & 0x1FFFFFFFULL) << 32);
}

// any v < 2^63  ->  v mod p
__device__ __forceinline__ uint64_t full61(uint64_t v) {
    v = (v & SKH_P) + (v >> 61);   // < 2^61 + 4 < 2p
    return v >= SKH_P ? v - SKH_P : v;
}

// H3: xi(x) = +1 iff ((a3 x + a2) x + a1) x + a0 mod p is odd.  s = {a0,a1,a2,a3,...}
// NARROW = true requires x < 2^32 (lazy 64x32 Horner, one final reduction); callers pick
// the variant once per loop, so the two paths are never if-converted into one.
template <bool NARROW>
__device__ __forceinline__ int xi_sign61_t(const uint64_t *s, uint64_t x) {
    if (NARROW) {
        // each step stays < 2^62 + 2^35 + 8 + 2^61 < 2^63
        uint64_t v = mulmod61_x32(s[3], (uint32_t)x) + s[2];
        v = mulmod61_x32(v, (uint32_t)x) + s[1];
        v = mulmod61_x32(v, (uint32_t)x) + s[0];
        return (full61(v) & 1ULL) ? 1 : -1;
    }
    uint64_t v = s[3];
    v = red61(mulmod61(v, x) + s[2]);
    v = red61(mulmod61(v, x) + s[1]);
    v = red61(mulmod61(v, x) + s[0]);
    return (v & 1ULL) ? 1 : -1;
}

// H4: g(x) = (b1 x + b0) mod p; the bucket is g mod w = g & (w-1).
template <bool NARROW>
__device__ __forceinline__ uint64_t hash_g61_t(uint64_t b0, uint64_t b1, uint64_t x) {
    if (NARROW) return full61(mulmod61_x32(b1, (uint32_t)x) + b0);
    return red61(mulmod61(b1, x) + b0);
}

// any key
__device__ __forceinline__ int xi_sign61(const uint64_t *s, uint64_t x) {
    return x < (1ULL << 32) ? xi_sign61_t<true>(s, x) : xi_sign61_t<false>(s, x);
}
__device__ __forceinline__ uint64_t hash_g61(uint64_t b0, uint64_t b1, uint64_t x) {
    return x < (1ULL << 32) ? hash_g61_t<true>(b0, b1, x) : hash_g61_t<false>(b0, b1, x);
}
