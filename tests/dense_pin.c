/* dense_pin.c — test-side dense evaluation of C3 sub-plan estimates at full sketch width,
 * used to pin the oracle's message-passing contraction (oracle/compass_oracle.c
 * or_contract_row) at w = 4096.  Independent of the oracle: it never
 * sorts, never uses the min-abs contraction identity; it materialises merged views
 * (m(l, r) = l if |l| <= |r| else r, left fold) and sums products over
 * bucket assignments, factored only by distributivity (a sum over one edge's buckets is
 * taken innermost).  Compiled by tests/test_oracle_fullwidth.py; test infrastructure only.
 *
 * Values must be small (|v| <= 1000) so that int64 inner sums are exact; the outer sums are
 * __int128.
 */
#include <stdint.h>
#include <stdlib.h>

static inline uint64_t uabs(int64_t v) { return v < 0 ? (uint64_t)(-v) : (uint64_t)v; }
static inline int64_t m2(int64_t l, int64_t r) { return uabs(l) <= uabs(r) ? l : r; }

/* out[a][b] = sum_i x[i] * fold(v0[.], v1[.], v2[.]) with constituent q indexed by i and
 * the other two (in order) by a and b.  Cost w^3. */
void dp_merged3_contract(const int64_t *v0, const int64_t *v1, const int64_t *v2, int q, const int64_t *x,
                         int64_t w, int64_t *out) {
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t a = 0; a < w; ++a) {
        for (int64_t b = 0; b < w; ++b) {
            int64_t acc = 0;
            if (q == 0) {        /* fold(v0[i], v1[a], v2[b]) */
                const int64_t va = v1[a], vb = v2[b];
                for (int64_t i = 0; i < w; ++i) acc += x[i] * m2(m2(v0[i], va), vb);
            } else if (q == 1) { /* fold(v0[a], v1[i], v2[b]) */
                const int64_t va = v0[a], vb = v2[b];
                for (int64_t i = 0; i < w; ++i) acc += x[i] * m2(m2(va, v1[i]), vb);
            } else {             /* fold(v0[a], v1[b], v2[i]) */
                const int64_t p = m2(v0[a], v1[b]);
                for (int64_t i = 0; i < w; ++i) acc += x[i] * m2(p, v2[i]);
            }
            out[a * w + b] = acc;
        }
    }
}

/* M[a][b] = m(u[a], v[b]) (two-constituent merged view, u first in canonical order) */
void dp_merged2(const int64_t *u, const int64_t *v, int64_t w, int64_t *M) {
#pragma omp parallel for
    for (int64_t a = 0; a < w; ++a)
        for (int64_t b = 0; b < w; ++b) M[a * w + b] = m2(u[a], v[b]);
}

/* sum_{l, j2, j3} A[l][j2] * B[j3][j2] * C[l][j3]  (three w x w int64 tensors on a triangle
 * of edges), as (lo, hi) of an __int128.  Inner sum over j2 in int64 (|A B| small enough for
 * the callers' value ranges), outer sums in __int128.  Cost w^3. */
void dp_triangle(const int64_t *A, const int64_t *B, const int64_t *C, int64_t w, int64_t *lohi) {
    __int128 total = 0;
#pragma omp parallel
    {
        __int128 part = 0;
#pragma omp for schedule(dynamic, 8)
        for (int64_t l = 0; l < w; ++l) {
            const int64_t *Al = A + l * w;
            for (int64_t j3 = 0; j3 < w; ++j3) {
                const int64_t *Bj = B + j3 * w;
                int64_t s = 0;
                for (int64_t j2 = 0; j2 < w; ++j2) s += Al[j2] * Bj[j2];
                part += (__int128)s * C[l * w + j3];
            }
        }
#pragma omp critical
        total += part;
    }
    lohi[0] = (int64_t)(uint64_t)total;
    lohi[1] = (int64_t)(total >> 64);
}
