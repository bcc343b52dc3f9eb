/*
 * compass_oracle.c — CPU ORACLE for the COMPASS Fast-AGMS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or execute anything under
 * oracle/.  The product path (paper_2102_02440_b200/) never does, and this file
 * shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C11.  Every function cites the passage of
 * /root/reference/PAPER.md ("PAPER.md:L") or SPEC.md ("SPEC.md:L") it follows,
 * and SURVEY.md §8(c) readings (H1-H6, O1-O10) where the paper is silent.
 *
 * Arithmetic:
 *   - hashing: exact arithmetic mod p = 2^61-1 via unsigned __int128 and '%'.
 *   - counters: int64 (O2/O3).
 *   - estimates: exact signed big integers (sign-magnitude, 32-bit limbs, fixed
 *     capacity, every overflow detected and reported), converted to double once,
 *     round-to-nearest-even (reading R13).
 *
 * Pins: tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <math.h>

/* ------------------------------------------------------------------------- */
/* H1-H4: hash family and seeds
 * The paper leaves the generators unspecified ("aspects that require careful
 * implementation"); SURVEY.md §8(c) H1-H4 fixes them.           */
/* ------------------------------------------------------------------------- */

#define OR_P ((uint64_t)0x1FFFFFFFFFFFFFFFULL) /* 2^61 - 1 */

static uint64_t mulmod_p(uint64_t a, uint64_t b) {
    unsigned __int128 t = (unsigned __int128)a * (unsigned __int128)b;
    return (uint64_t)(t % OR_P);
}
static uint64_t addmod_p(uint64_t a, uint64_t b) {
    unsigned __int128 t = (unsigned __int128)a + (unsigned __int128)b;
    return (uint64_t)(t % OR_P);
}

/* H2 mixer: splitmix64 finalizer ("splitmix-style finalizer"). */
uint64_t or_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* H2 string hash: FNV-1a 64 over the canonical edge id bytes. */
uint64_t or_fnv1a64(const char *s) {
    uint64_t h = 0xCBF29CE484222325ULL;
    for (const unsigned char *p = (const unsigned char *)s; *p; ++p) {
        h ^= (uint64_t)(*p);
        h *= 0x100000001B3ULL;
    }
    return h;
}

/* H2 coefficient c(master, edge, row, role, i); role 0 = xi (i=0..3), 1 = h (i=0..1).
 * Both endpoints of an edge derive identical seeds ("share the same
 * family"), different edges different seeds (PAPER.md:99 two independent sketches). */
uint64_t or_coef(uint64_t master, const char *edge_id, uint32_t row, uint32_t role, uint32_t idx) {
    uint64_t inner = or_splitmix64(((uint64_t)row << 8) | ((uint64_t)role << 4) | (uint64_t)idx);
    uint64_t mid = or_splitmix64(or_fnv1a64(edge_id) ^ inner);
    return or_splitmix64(master ^ mid) % OR_P;
}

/* H1: key canonicalisation.  Sign-extend to int64, reinterpret as uint64, reduce mod p. */
uint64_t or_canon(int64_t key) {
    return ((uint64_t)key) % OR_P;
}

/* H3: xi = +1 if ((a3 x + a2) x + a1) x + a0 mod p is odd, else -1. */
static int xi_eval(const uint64_t a[4], uint64_t x) {
    uint64_t v = a[3];
    v = addmod_p(mulmod_p(v, x), a[2]);
    v = addmod_p(mulmod_p(v, x), a[1]);
    v = addmod_p(mulmod_p(v, x), a[0]);
    return (v & 1ULL) ? +1 : -1;
}

/* H4: g = (b1 x + b0) mod p; bucket = g mod w. */
static uint64_t g_eval(const uint64_t b[2], uint64_t x) {
    return addmod_p(mulmod_p(b[1], x), b[0]);
}

typedef struct { uint64_t a[4]; uint64_t b[2]; } row_seed;

static void derive_row_seed(uint64_t master, const char *edge, uint32_t r, row_seed *s) {
    for (uint32_t i = 0; i < 4; ++i) s->a[i] = or_coef(master, edge, r, 0, i);
    for (uint32_t i = 0; i < 2; ++i) s->b[i] = or_coef(master, edge, r, 1, i);
}

int or_xi(uint64_t master, const char *edge, uint32_t row, int64_t key) {
    row_seed s; derive_row_seed(master, edge, row, &s);
    return xi_eval(s.a, or_canon(key));
}

uint64_t or_bucket(uint64_t master, const char *edge, uint32_t row, int64_t key, uint64_t w) {
    row_seed s; derive_row_seed(master, edge, row, &s);
    return g_eval(s.b, or_canon(key)) % w;
}

/* ------------------------------------------------------------------------- */
/* O1: push-down selection ("computes the exact selectivity
 * cardinalities"; kinds point/range/subset PAPER.md:173).  Conjunction;
 * ranges inclusive [lo, hi] (SURVEY.md §8(c) reading 11).                    */
/* ------------------------------------------------------------------------- */

enum { OR_POINT = 0, OR_RANGE = 1, OR_SUBSET = 2 };

static int64_t col_value(const void *col, int is64, int64_t i) {
    return is64 ? ((const int64_t *)col)[i] : (int64_t)((const int32_t *)col)[i];
}

static int cmp_i64(const void *x, const void *y) {
    int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    return (a > b) - (a < b);
}

/* mask[i] = AND of predicates; returns popcount(mask) = exact survivors. */
int64_t or_filter(int64_t n_rows, const void *const *cols, const int *col_is64,
                  int n_pred, const int *pred_col, const int *pred_kind,
                  const int64_t *pred_lo, const int64_t *pred_hi,
                  const int64_t *const *pred_set, const int64_t *pred_set_n,
                  uint8_t *mask) {
    /* sorted copies of subset sets, for bsearch (a library primitive as a step) */
    int64_t **sets = (int64_t **)calloc((size_t)(n_pred > 0 ? n_pred : 1), sizeof(int64_t *));
    for (int p = 0; p < n_pred; ++p) {
        if (pred_kind[p] == OR_SUBSET && pred_set_n[p] > 0) {
            sets[p] = (int64_t *)malloc((size_t)pred_set_n[p] * sizeof(int64_t));
            memcpy(sets[p], pred_set[p], (size_t)pred_set_n[p] * sizeof(int64_t));
            qsort(sets[p], (size_t)pred_set_n[p], sizeof(int64_t), cmp_i64);
        }
    }
    int64_t count = 0;
    for (int64_t i = 0; i < n_rows; ++i) {
        int keep = 1;
        for (int p = 0; p < n_pred && keep; ++p) {
            int64_t v = col_value(cols[pred_col[p]], col_is64[pred_col[p]], i);
            if (pred_kind[p] == OR_POINT) keep = (v == pred_lo[p]);
            else if (pred_kind[p] == OR_RANGE) keep = (pred_lo[p] <= v && v <= pred_hi[p]);
            else keep = (pred_set_n[p] > 0) &&
                        bsearch(&v, sets[p], (size_t)pred_set_n[p], sizeof(int64_t), cmp_i64) != NULL;
        }
        mask[i] = (uint8_t)keep;
        count += keep;
    }
    for (int p = 0; p < n_pred; ++p) free(sets[p]);
    free(sets);
    return count;
}

/* ------------------------------------------------------------------------- */
/* O2 / O3: Fast-AGMS build, tuple by tuple.
 *   1-D: sk[r][h_r(x)] += xi_r(x).
 *   2-D partitioned: M[r][h^e_r(x)][h^f_r(y)] += xi^e_r(x) xi^f_r(y),
 *   dim 0 = the canonically first edge.
 * Adds into `out` (int64, [d][w0] or [d][w0][w1]); rows with mask[i]==0 skipped.
 * Returns 0, or -1 on invalid arguments.                                      */
/* ------------------------------------------------------------------------- */
int or_build(int64_t n_rows, const uint8_t *mask,
             const void *key0, int key0_is64, const void *key1, int key1_is64,
             int d, int ndim, const int64_t *w, const char *edge0, const char *edge1,
             uint64_t master, int64_t *out) {
    if (d < 1 || (ndim != 1 && ndim != 2)) return -1;
    row_seed *s0 = (row_seed *)malloc((size_t)d * sizeof(row_seed));
    row_seed *s1 = (row_seed *)malloc((size_t)d * sizeof(row_seed));
    for (int r = 0; r < d; ++r) {
        derive_row_seed(master, edge0, (uint32_t)r, &s0[r]);
        if (ndim == 2) derive_row_seed(master, edge1, (uint32_t)r, &s1[r]);
    }
    int64_t cells = (ndim == 1) ? w[0] : w[0] * w[1];
    for (int64_t i = 0; i < n_rows; ++i) {
        if (mask && !mask[i]) continue;
        uint64_t x = or_canon(col_value(key0, key0_is64, i));
        uint64_t y = (ndim == 2) ? or_canon(col_value(key1, key1_is64, i)) : 0;
        for (int r = 0; r < d; ++r) {
            int64_t j0 = (int64_t)(g_eval(s0[r].b, x) % (uint64_t)w[0]);
            int sign = xi_eval(s0[r].a, x);
            int64_t cell = j0;
            if (ndim == 2) {
                int64_t j1 = (int64_t)(g_eval(s1[r].b, y) % (uint64_t)w[1]);
                sign *= xi_eval(s1[r].a, y);
                cell = j0 * w[1] + j1;
            }
            out[(int64_t)r * cells + cell] += sign;
        }
    }
    free(s0); free(s1);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O3' (n-D partitioned tensor, "a table with 3 joins has a 3-D tensor
 * as its sketch, with one dimension for every join attribute"): for every surviving
 * tuple and row r, the cell [h^{e_0}_r(x_0)]..[h^{e_{n-1}}_r(x_{n-1})] gets
 * prod_q xi^{e_q}_r(x_q); dims in canonical edge order (SURVEY.md H6 generalised).
 * keys[q] / key_is64[q] / edges[q] / w[q] per dimension, 1 <= ndim <= 3; adds into
 * `out` (int64, [d][w_0]..[w_{ndim-1}], row-major).  Returns 0, or -1.        */
/* ------------------------------------------------------------------------- */
int or_build_nd(int64_t n_rows, const uint8_t *mask, int ndim, const void *const *keys, const int *key_is64,
                int d, const int64_t *w, const char *const *edges, uint64_t master, int64_t *out) {
    if (d < 1 || ndim < 1 || ndim > 3) return -1;
    row_seed *s = (row_seed *)malloc((size_t)d * 3 * sizeof(row_seed));
    for (int q = 0; q < ndim; ++q)
        for (int r = 0; r < d; ++r) derive_row_seed(master, edges[q], (uint32_t)r, &s[q * d + r]);
    int64_t cells = 1;
    for (int q = 0; q < ndim; ++q) cells *= w[q];
    for (int64_t i = 0; i < n_rows; ++i) {
        if (mask && !mask[i]) continue;
        for (int r = 0; r < d; ++r) {
            int64_t cell = 0;
            int sign = 1;
            for (int q = 0; q < ndim; ++q) {
                uint64_t x = or_canon(col_value(keys[q], key_is64[q], i));
                cell = cell * w[q] + (int64_t)(g_eval(s[q * d + r].b, x) % (uint64_t)w[q]);
                sign *= xi_eval(s[q * d + r].a, x);
            }
            out[(int64_t)r * cells + cell] += sign;
        }
    }
    free(s);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Exact signed big integers (sign-magnitude, BN_L x 32-bit limbs).            */
/* ------------------------------------------------------------------------- */

#define BN_L 16 /* 512 bits of magnitude */

typedef struct { int neg; int n; uint32_t m[BN_L]; } bn;

static int bn_overflow = 0; /* set on any overflow; checked by the entry points */

static void bn_zero(bn *a) { a->neg = 0; a->n = 0; }

static void bn_norm(bn *a) {
    while (a->n > 0 && a->m[a->n - 1] == 0) a->n--;
    if (a->n == 0) a->neg = 0;
}

static void bn_from_i64(bn *a, int64_t v) {
    uint64_t mag = (v < 0) ? (uint64_t)(-(v + 1)) + 1ULL : (uint64_t)v;
    a->neg = v < 0;
    a->m[0] = (uint32_t)mag;
    a->m[1] = (uint32_t)(mag >> 32);
    a->n = 2;
    bn_norm(a);
}

static int mag_cmp(const bn *a, const bn *b) {
    if (a->n != b->n) return a->n < b->n ? -1 : 1;
    for (int i = a->n - 1; i >= 0; --i)
        if (a->m[i] != b->m[i]) return a->m[i] < b->m[i] ? -1 : 1;
    return 0;
}

/* r = |a| + |b| (magnitudes) */
static void mag_add(bn *r, const bn *a, const bn *b) {
    int n = a->n > b->n ? a->n : b->n;
    uint64_t carry = 0;
    bn t;
    for (int i = 0; i < n; ++i) {
        uint64_t s = carry;
        if (i < a->n) s += a->m[i];
        if (i < b->n) s += b->m[i];
        t.m[i] = (uint32_t)s;
        carry = s >> 32;
    }
    t.n = n;
    if (carry) {
        if (n >= BN_L) { bn_overflow = 1; t.n = n; }
        else { t.m[n] = (uint32_t)carry; t.n = n + 1; }
    }
    t.neg = 0;
    *r = t;
}

/* r = |a| - |b|, requires |a| >= |b| */
static void mag_sub(bn *r, const bn *a, const bn *b) {
    int64_t borrow = 0;
    bn t;
    for (int i = 0; i < a->n; ++i) {
        int64_t s = (int64_t)a->m[i] - borrow - (i < b->n ? (int64_t)b->m[i] : 0);
        borrow = s < 0;
        if (s < 0) s += ((int64_t)1 << 32);
        t.m[i] = (uint32_t)s;
    }
    t.n = a->n;
    t.neg = 0;
    bn_norm(&t);
    *r = t;
}

static void bn_add(bn *r, const bn *a, const bn *b) {
    if (a->n == 0) { *r = *b; return; }
    if (b->n == 0) { *r = *a; return; }
    if (a->neg == b->neg) {
        int neg = a->neg;
        mag_add(r, a, b);
        r->neg = neg;
    } else {
        int c = mag_cmp(a, b);
        if (c == 0) { bn_zero(r); return; }
        int neg = (c > 0) ? a->neg : b->neg;
        if (c > 0) mag_sub(r, a, b); else mag_sub(r, b, a);
        r->neg = neg;
    }
    bn_norm(r);
}

static void bn_sub(bn *r, const bn *a, const bn *b) {
    bn nb = *b;
    if (nb.n) nb.neg = !nb.neg;
    bn_add(r, a, &nb);
}

static void bn_mul(bn *r, const bn *a, const bn *b) {
    if (a->n == 0 || b->n == 0) { bn_zero(r); return; }
    if (a->n + b->n > BN_L + 1) { bn_overflow = 1; bn_zero(r); return; }
    uint32_t t[2 * BN_L + 2];
    memset(t, 0, sizeof(t));
    for (int i = 0; i < a->n; ++i) {
        uint64_t carry = 0;
        for (int j = 0; j < b->n; ++j) {
            uint64_t cur = (uint64_t)a->m[i] * b->m[j] + t[i + j] + carry;
            t[i + j] = (uint32_t)cur;
            carry = cur >> 32;
        }
        t[i + b->n] = (uint32_t)carry;
    }
    int n = a->n + b->n;
    while (n > 0 && t[n - 1] == 0) n--;
    if (n > BN_L) { bn_overflow = 1; bn_zero(r); return; }
    bn out;
    out.n = n;
    memcpy(out.m, t, (size_t)n * sizeof(uint32_t));
    out.neg = a->neg ^ b->neg;
    bn_norm(&out);
    *r = out;
}

static void bn_mul_i64(bn *r, const bn *a, int64_t v) {
    bn b; bn_from_i64(&b, v);
    bn_mul(r, a, &b);
}

/* acc += a * b */
static void bn_addmul(bn *acc, const bn *a, const bn *b) {
    bn t; bn_mul(&t, a, b); bn_add(acc, acc, &t);
}

/* Correctly rounded (nearest, ties-to-even) conversion to double. */
static double bn_to_double(const bn *a) {
    if (a->n == 0) return 0.0;
    int top = a->n - 1;
    int hb = 31; while (!((a->m[top] >> hb) & 1u)) hb--;
    int nbits = top * 32 + hb + 1;
    double mag;
    if (nbits <= 64) {
        uint64_t v = a->m[0] | ((a->n > 1) ? ((uint64_t)a->m[1] << 32) : 0);
        if (nbits <= 53) mag = (double)v;
        else {
            int sh = nbits - 53;
            uint64_t keep = v >> sh, rem = v & ((1ULL << sh) - 1), half = 1ULL << (sh - 1);
            if (rem > half || (rem == half && (keep & 1ULL))) keep++;
            mag = ldexp((double)keep, sh);
        }
    } else {
        /* extract bits [nbits-64, nbits) as `w`, sticky = any lower bit set */
        int lo = nbits - 64;
        uint64_t w = 0;
        for (int b = 0; b < 64; ++b) {
            int bit = lo + b;
            if ((a->m[bit / 32] >> (bit % 32)) & 1u) w |= (1ULL << b);
        }
        int sticky = 0;
        for (int bit = 0; bit < lo && !sticky; ++bit)
            if ((a->m[bit / 32] >> (bit % 32)) & 1u) sticky = 1;
        uint64_t keep = w >> 11, rem = w & 0x7FFULL;
        if (rem > 0x400ULL || (rem == 0x400ULL && (sticky || (keep & 1ULL)))) keep++;
        mag = ldexp((double)keep, lo + 11);
    }
    return a->neg ? -mag : mag;
}

/* decimal string; returns length or -1 if buffer too small */
static int bn_to_dec(const bn *a, char *out, int out_len) {
    if (a->n == 0) { if (out_len < 2) return -1; out[0] = '0'; out[1] = 0; return 1; }
    bn t = *a;
    char buf[200];
    int len = 0;
    while (t.n > 0) {
        uint64_t rem = 0;
        for (int i = t.n - 1; i >= 0; --i) {
            uint64_t cur = (rem << 32) | t.m[i];
            t.m[i] = (uint32_t)(cur / 1000000000ULL);
            rem = cur % 1000000000ULL;
        }
        while (t.n > 0 && t.m[t.n - 1] == 0) t.n--;
        for (int k = 0; k < 9; ++k) { buf[len++] = (char)('0' + rem % 10); rem /= 10; }
    }
    while (len > 1 && buf[len - 1] == '0') len--;
    int pos = 0;
    if (a->neg) { if (pos >= out_len - 1) return -1; out[pos++] = '-'; }
    if (pos + len >= out_len) return -1;
    for (int i = len - 1; i >= 0; --i) out[pos++] = buf[i];
    out[pos] = 0;
    return pos;
}

/* exported helpers, pinned against Python's exact int / float(int) */
int or_bn_selftest_mul_add(int n, const int64_t *xs, const int64_t *ys, char *out, int out_len) {
    /* returns decimal of sum_i xs[i]*ys[i]*xs[i]  (exercises multi-limb products) */
    bn acc; bn_zero(&acc);
    bn_overflow = 0;
    for (int i = 0; i < n; ++i) {
        bn a, b, t;
        bn_from_i64(&a, xs[i]); bn_from_i64(&b, ys[i]);
        bn_mul(&t, &a, &b); bn_mul(&t, &t, &a);
        bn_add(&acc, &acc, &t);
    }
    if (bn_overflow) return -2;
    return bn_to_dec(&acc, out, out_len);
}

double or_bn_selftest_to_double(int n, const int64_t *xs) {
    /* product of xs as big integer, converted once */
    bn acc; bn_from_i64(&acc, 1);
    bn_overflow = 0;
    for (int i = 0; i < n; ++i) bn_mul_i64(&acc, &acc, xs[i]);
    return bn_to_double(&acc);
}

/* ------------------------------------------------------------------------- */
/* O6 / O7: sub-plan estimate for ONE sketch row.
 *
 * The sub-plan is given as a tensor network: tables
 * t = 0..T-1, edges e = 0..E-1 (passed in canonical edge-id order), bucket
 * count w_e per edge (vectors already folded, O5).  Each table contributes:
 *   kind 0 VEC    : 1 leg, data[3t] int64[w_leg]            (1-D sketch)
 *   kind 1 MAT    : 2 legs, data[3t] int64[w_l0 * w_l1]     (partitioned)
 *   kind 2 MERGED : k<=3 legs (canonical order), data[3t+q] = constituent q's 1-D
 *                   sketch; entry = left fold of the min-abs rule,
 *                   i.e. the first constituent of minimal |value|.
 * E_r = sum over all assignments of a bucket to every edge of prod_t T_t(...).
 *
 * or_contract_brute_row : that definition, enumerated literally (tiny w only).
 * or_contract_row       : the same number by exact message passing on the
 *                         network (tree; a single cycle is conditioned on one
 *                         edge), with the min-abs contraction identity of
 *                         SURVEY.md §8(c) O9 for merged tables.  Pinned to
 *                         or_contract_brute_row (tests P5).
 * Both return the exact value as a decimal string (and via *out_dbl rounded).
 * Return: >=0 ok, -1 bad arguments, -2 overflow, -3 unsupported (>1 cycle).
 */
/* ------------------------------------------------------------------------- */

enum { K_VEC = 0, K_MAT = 1, K_MERGED = 2, K_TEN3 = 3 };   /* K_TEN3: 3-D partitioned tensor */

typedef struct {
    int T, E;
    const int *kind, *nlegs, *legs;          /* legs[3t + q] */
    const int64_t *const *data;              /* data[3t + q] */
    const int64_t *w;                        /* w[e] */
    int ends[64][2];                         /* table endpoints of each edge */
} net;

static uint64_t uabs64(int64_t v) { return v < 0 ? (uint64_t)(-(v + 1)) + 1ULL : (uint64_t)v; }

/* left fold of the min-abs rule over constituent values, in order:
 * m(l, r) = l if |l| <= |r| else r. */
static int64_t fold_minabs(const int64_t *vals, int k) {
    int64_t acc = vals[0];
    for (int q = 1; q < k; ++q)
        if (!(uabs64(acc) <= uabs64(vals[q]))) acc = vals[q];
    return acc;
}

/* T_t evaluated at per-leg indices idx[q] */
static int64_t tensor_at(const net *g, int t, const int64_t *idx) {
    int k = g->nlegs[t];
    const int *lg = &g->legs[3 * t];
    if (g->kind[t] == K_VEC) return g->data[3 * t][idx[0]];
    if (g->kind[t] == K_MAT) return g->data[3 * t][idx[0] * g->w[lg[1]] + idx[1]];
    if (g->kind[t] == K_TEN3) return g->data[3 * t][(idx[0] * g->w[lg[1]] + idx[1]) * g->w[lg[2]] + idx[2]];
    int64_t vals[3] = {0, 0, 0};
    for (int q = 0; q < k; ++q) vals[q] = g->data[3 * t + q][idx[q]];
    return fold_minabs(vals, k);
}

static int net_init(net *g, int T, const int *kind, const int *nlegs, const int *legs,
                    const int64_t *const *data, int E, const int64_t *w) {
    if (T < 1 || E < 0 || E > 64) return -1;
    g->T = T; g->E = E; g->kind = kind; g->nlegs = nlegs; g->legs = legs; g->data = data; g->w = w;
    int cnt[64] = {0};
    for (int t = 0; t < T; ++t) {
        if (nlegs[t] < 1 || nlegs[t] > 3) return -1;
        if (kind[t] == K_VEC && nlegs[t] != 1) return -1;
        if (kind[t] == K_MAT && nlegs[t] != 2) return -1;
        if (kind[t] == K_TEN3 && nlegs[t] != 3) return -1;
        for (int q = 0; q < nlegs[t]; ++q) {
            int e = legs[3 * t + q];
            if (e < 0 || e >= E || cnt[e] >= 2) return -1;
            g->ends[e][cnt[e]++] = t;
        }
    }
    for (int e = 0; e < E; ++e) if (cnt[e] != 2) return -1;
    return 0;
}

/* --- literal definition ---------------------------------------------------- */
static int contract_brute(const net *g, bn *out) {
    double total = 1;
    for (int e = 0; e < g->E; ++e) total *= (double)g->w[e];
    if (total > 5e8) return -1;
    int64_t asg[64] = {0};
    bn acc; bn_zero(&acc);
    for (;;) {
        bn prod; bn_from_i64(&prod, 1);
        for (int t = 0; t < g->T; ++t) {
            int64_t idx[3];
            for (int q = 0; q < g->nlegs[t]; ++q) idx[q] = asg[g->legs[3 * t + q]];
            bn_mul_i64(&prod, &prod, tensor_at(g, t, idx));
            if (prod.n == 0) break;
        }
        bn_add(&acc, &acc, &prod);
        int e = 0;
        while (e < g->E) { if (++asg[e] < g->w[e]) break; asg[e] = 0; ++e; }
        if (e == g->E) break;
    }
    *out = acc;
    return 0;
}

/* --- message passing ------------------------------------------------------- */

typedef struct {
    const net *g;
    int cond_edge;        /* conditioned edge (-1: none) */
    int64_t cond_val;     /* its bucket */
    bn *msg[64];          /* msg[e]: vector over edge e sent from child to parent */
} mp_ctx;

/* #{i : s[i] < t} */
static int64_t lower_bound_u64(const uint64_t *s, int64_t n, uint64_t t) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (s[mid] < t) lo = mid + 1; else hi = mid; }
    return lo;
}
/* #{i : s[i] <= t} */
static int64_t upper_bound_u64(const uint64_t *s, int64_t n, uint64_t t) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (s[mid] <= t) lo = mid + 1; else hi = mid; }
    return lo;
}

typedef struct { uint64_t key; int64_t idx; } kv;
static int cmp_kv(const void *x, const void *y) {
    const kv *a = (const kv *)x, *b = (const kv *)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

/* Node t, parent edge p (-1 = root). Children edges: tree edges at t other than p.
 * Writes message over p into ctx->msg[p] (allocated by caller), or scalar into *root_out. */
static int node_eval(mp_ctx *c, int t, int p, bn *root_out);

static int dfs(mp_ctx *c, int t, int p) {
    const net *g = c->g;
    for (int q = 0; q < g->nlegs[t]; ++q) {
        int e = g->legs[3 * t + q];
        if (e == p || e == c->cond_edge) continue;
        int child = g->ends[e][0] == t ? g->ends[e][1] : g->ends[e][0];
        int rc = dfs(c, child, e);
        if (rc) return rc;
    }
    if (p >= 0) return node_eval(c, t, p, NULL);
    return 0;
}

static int node_eval(mp_ctx *c, int t, int p, bn *root_out) {
    const net *g = c->g;
    int k = g->nlegs[t];
    const int *lg = &g->legs[3 * t];
    int role[3];             /* 0 child, 1 parent, 2 fixed */
    int nchild = 0, child_q[3];
    for (int q = 0; q < k; ++q) {
        if (lg[q] == c->cond_edge) role[q] = 2;
        else if (lg[q] == p) role[q] = 1;
        else { role[q] = 0; child_q[nchild++] = q; }
    }
    bn *out = (p >= 0) ? c->msg[p] : NULL;
    if (out) for (int64_t j = 0; j < g->w[p]; ++j) bn_zero(&out[j]);
    bn scalar; bn_zero(&scalar);

    if (g->kind[t] != K_MERGED || nchild == 0) {
        /* explicit loop over all free-leg index combinations (<= w^2 for VEC/MAT;
         * MERGED leaves have a single free leg) */
        int64_t idx[3] = {0, 0, 0};
        for (int q = 0; q < k; ++q) if (role[q] == 2) idx[q] = c->cond_val;
        for (;;) {
            bn term; bn_from_i64(&term, tensor_at(g, t, idx));
            for (int i = 0; i < nchild; ++i) {
                int q = child_q[i];
                bn_mul(&term, &term, &c->msg[lg[q]][idx[q]]);
            }
            if (out) {
                int qp = -1; for (int q = 0; q < k; ++q) if (role[q] == 1) qp = q;
                bn_add(&out[idx[qp]], &out[idx[qp]], &term);
            } else bn_add(&scalar, &scalar, &term);
            int q = 0;
            while (q < k) {
                if (role[q] != 2) { if (++idx[q] < g->w[lg[q]]) break; idx[q] = 0; }
                ++q;
            }
            if (q == k) break;
        }
    } else {
        /* MERGED with >=1 child: contract child leg qc with the O9 identity,
         * iterate explicitly over the remaining free legs. */
        int qc = child_q[0];
        int eq = lg[qc];
        int64_t wq = g->w[eq];
        const int64_t *cq = g->data[3 * t + qc];
        const bn *x = c->msg[eq];
        kv *ord = (kv *)malloc((size_t)wq * sizeof(kv));
        for (int64_t i = 0; i < wq; ++i) { ord[i].key = uabs64(cq[i]); ord[i].idx = i; }
        qsort(ord, (size_t)wq, sizeof(kv), cmp_kv);
        uint64_t *sabs = (uint64_t *)malloc((size_t)wq * sizeof(uint64_t));
        bn *P1 = (bn *)malloc((size_t)(wq + 1) * sizeof(bn));   /* prefix sums of x   */
        bn *P2 = (bn *)malloc((size_t)(wq + 1) * sizeof(bn));   /* prefix sums of x*c */
        bn_zero(&P1[0]); bn_zero(&P2[0]);
        for (int64_t s = 0; s < wq; ++s) {
            sabs[s] = ord[s].key;
            bn xc; bn_mul_i64(&xc, &x[ord[s].idx], cq[ord[s].idx]);
            bn_add(&P1[s + 1], &P1[s], &x[ord[s].idx]);
            bn_add(&P2[s + 1], &P2[s], &xc);
        }
        int64_t idx[3] = {0, 0, 0};
        for (int q = 0; q < k; ++q) if (role[q] == 2) idx[q] = c->cond_val;
        for (;;) {
            /* L = fold of constituents before qc, R = fold of those after qc */
            int64_t vals[3]; int nl = 0, nr = 0; int64_t lv[3] = {0, 0, 0}, rv[3] = {0, 0, 0};
            for (int q = 0; q < k; ++q) {
                if (q == qc) continue;
                vals[q] = g->data[3 * t + q][idx[q]];
                if (q < qc) lv[nl++] = vals[q]; else rv[nr++] = vals[q];
            }
            bn V; bn_zero(&V);
            bn tmp;
            if (nl > 0) {
                int64_t L = fold_minabs(lv, nl);
                uint64_t aL = uabs64(L);
                int64_t nless = lower_bound_u64(sabs, wq, aL);         /* |c| < |L| */
                int64_t win = L;
                if (nr > 0) { int64_t R = fold_minabs(rv, nr); if (!(aL <= uabs64(R))) win = R; }
                /* A = {|c| >= |L|}: value m(L,R) */
                bn sA; bn_sub(&sA, &P1[wq], &P1[nless]);
                bn_mul_i64(&tmp, &sA, win); bn_add(&V, &V, &tmp);
                int64_t endB = nless;
                if (nr > 0) {
                    int64_t R = fold_minabs(rv, nr);
                    int64_t nle = upper_bound_u64(sabs, wq, uabs64(R));  /* |c| <= |R| */
                    if (nle < endB) {
                        /* C = {|R| < |c| < |L|}: value R */
                        bn sC; bn_sub(&sC, &P1[endB], &P1[nle]);
                        bn_mul_i64(&tmp, &sC, R); bn_add(&V, &V, &tmp);
                        endB = nle;
                    }
                }
                /* B = {|c| < |L|, |c| <= |R|}: value c itself */
                bn_add(&V, &V, &P2[endB]);
            } else {
                int64_t R = fold_minabs(rv, nr);
                int64_t nle = upper_bound_u64(sabs, wq, uabs64(R));
                bn sC; bn_sub(&sC, &P1[wq], &P1[nle]);
                bn_mul_i64(&tmp, &sC, R); bn_add(&V, &V, &tmp);
                bn_add(&V, &V, &P2[nle]);
            }
            for (int i = 1; i < nchild; ++i) {
                int q = child_q[i];
                bn_mul(&V, &V, &c->msg[lg[q]][idx[q]]);
            }
            if (out) {
                int qp = -1; for (int q = 0; q < k; ++q) if (role[q] == 1) qp = q;
                bn_add(&out[idx[qp]], &out[idx[qp]], &V);
            } else bn_add(&scalar, &scalar, &V);
            int q = 0;
            while (q < k) {
                if (role[q] != 2 && q != qc) { if (++idx[q] < g->w[lg[q]]) break; idx[q] = 0; }
                ++q;
            }
            if (q == k) break;
        }
        free(ord); free(sabs); free(P1); free(P2);
    }
    if (!out && root_out) *root_out = scalar;
    return 0;
}

/* is edge e on a cycle? (removing it keeps the network connected) */
static int edge_on_cycle(const net *g, int e) {
    int seen[64] = {0}, stack[64], sp = 0;
    seen[0] = 1; stack[sp++] = 0;
    while (sp) {
        int t = stack[--sp];
        for (int q = 0; q < g->nlegs[t]; ++q) {
            int f = g->legs[3 * t + q];
            if (f == e) continue;
            int u = g->ends[f][0] == t ? g->ends[f][1] : g->ends[f][0];
            if (!seen[u]) { seen[u] = 1; stack[sp++] = u; }
        }
    }
    for (int t = 0; t < g->T; ++t) if (!seen[t]) return 0;
    return 1;
}

static int contract_mp(const net *g, bn *out) {
    int cyc = g->E - g->T + 1;
    if (cyc < 0) return -1;
    if (cyc > 1) return -3;
    mp_ctx c; memset(&c, 0, sizeof(c));
    c.g = g; c.cond_edge = -1;
    if (cyc == 1) {
        /* condition on the cycle edge whose endpoints have the most legs (ties: first) */
        int best = -1, bestdeg = -1;
        for (int e = 0; e < g->E; ++e) {
            if (!edge_on_cycle(g, e)) continue;
            int dg = g->nlegs[g->ends[e][0]] + g->nlegs[g->ends[e][1]];
            if (dg > bestdeg) { bestdeg = dg; best = e; }
        }
        if (best < 0) return -1;
        c.cond_edge = best;
    }
    for (int e = 0; e < g->E; ++e) c.msg[e] = (bn *)malloc((size_t)g->w[e] * sizeof(bn));
    bn acc; bn_zero(&acc);
    int64_t nb = (c.cond_edge >= 0) ? g->w[c.cond_edge] : 1;
    int rc = 0;
    for (int64_t b = 0; b < nb && rc == 0; ++b) {
        c.cond_val = b;
        rc = dfs(&c, 0, -1);
        if (rc) break;
        bn s; rc = node_eval(&c, 0, -1, &s);
        bn_add(&acc, &acc, &s);
    }
    for (int e = 0; e < g->E; ++e) free(c.msg[e]);
    *out = acc;
    return rc;
}

static int finish(int rc, const bn *v, char *out, int out_len, double *out_dbl) {
    if (rc) return rc;
    if (bn_overflow) return -2;
    if (out_dbl) *out_dbl = bn_to_double(v);
    if (out && bn_to_dec(v, out, out_len) < 0) return -1;
    return 0;
}

int or_contract_row(int T, const int *kind, const int *nlegs, const int *legs,
                    const int64_t *const *data, int E, const int64_t *w,
                    char *out, int out_len, double *out_dbl) {
    net g;
    if (net_init(&g, T, kind, nlegs, legs, data, E, w)) return -1;
    bn_overflow = 0;
    bn v; int rc = contract_mp(&g, &v);
    return finish(rc, &v, out, out_len, out_dbl);
}

int or_contract_brute_row(int T, const int *kind, const int *nlegs, const int *legs,
                          const int64_t *const *data, int E, const int64_t *w,
                          char *out, int out_len, double *out_dbl) {
    net g;
    if (net_init(&g, T, kind, nlegs, legs, data, E, w)) return -1;
    bn_overflow = 0;
    bn v; int rc = contract_brute(&g, &v);
    return finish(rc, &v, out, out_len, out_dbl);
}

/* O6 two-way, one row, exact: sum_j a[j] * b[j]. */
int or_two_way_row(int64_t w, const int64_t *a, const int64_t *b, char *out, int out_len, double *out_dbl) {
    bn acc; bn_zero(&acc);
    bn_overflow = 0;
    for (int64_t j = 0; j < w; ++j) {
        bn x, y; bn_from_i64(&x, a[j]); bn_from_i64(&y, b[j]);
        bn_addmul(&acc, &x, &y);
    }
    return finish(0, &acc, out, out_len, out_dbl);
}

/* median helper on decimal-free path: exact compare of two decimal strings is done
 * in Python; here we expose the to-double conversion of an exact decimal value. */
double or_dec_to_double(const char *s) {
    bn acc; bn_zero(&acc);
    bn ten; bn_from_i64(&ten, 10);
    int neg = 0;
    if (*s == '-') { neg = 1; ++s; }
    bn_overflow = 0;
    for (; *s; ++s) {
        bn d; bn_from_i64(&d, (int64_t)(*s - '0'));
        bn_mul(&acc, &acc, &ten);
        bn_add(&acc, &acc, &d);
    }
    if (neg && acc.n) acc.neg = 1;
    return bn_to_double(&acc);
}
