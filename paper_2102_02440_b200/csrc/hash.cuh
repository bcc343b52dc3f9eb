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

// H3: xi(x) = +1 iff ((a3 x + a2) x + a1) x + a0 mod p is odd.  s = {a0,a1,a2,a3,...}
__device__ __forceinline__ int xi_sign61(const uint64_t *s, uint64_t x) {
    uint64_t v = s[3];
    v = red61(mulmod61(v, x) + s[2]);
    v = red61(mulmod61(v, x) + s[1]);
    v = red61(mulmod61(v, x) + s[0]);
    return (v & 1ULL) ? 1 : -1;
}

// H4: g(x) = (b1 x + b0) mod p; the bucket is g mod w = g & (w-1).
__device__ __forceinline__ uint64_t hash_g61(uint64_t b0, uint64_t b1, uint64_t x) {
    return red61(mulmod61(b1, x) + b0);
}
