/*
 * compass_b200.h — C-ABI of the B200-native COMPASS hot path (arXiv 2102.02440).
 *
 * The data-parallel hot path of COMPASS: an online Fast-AGMS sketch build fused
 * with push-down selection, the merge of partial sketches, the sketch-composition
 * estimates of join cardinality and the greedy join-order enumerator that consumes
 * them.  Citations: PAPER.md / SPEC.md under /root/reference, SURVEY.md §8(b).
 *
 * Conventions (all entry points):
 *   - Plain C types only.  "device" pointers are CUDA device pointers on the
 *     sketch's device; "host" pointers are ordinary host memory.
 *   - Asynchronous entry points enqueue work on `stream` (a cudaStream_t passed
 *     as void*; NULL = legacy default stream) and return immediately.  Entry
 *     points that return host values (estimate_*, plan_greedy) synchronise
 *     `stream` before returning.
 *   - Ownership: columns, survivor counters and caller-provided counter buffers
 *     are owned by the caller and must stay valid until the stream work that
 *     uses them completes.  The library owns only what it allocated.
 *   - Errors: no exception crosses the ABI.  Every call returns an sk_status;
 *     sk_last_error() gives a thread-local message for the last failure.
 *   - Concurrency: a sketch must not be updated from two streams at once.
 *   - There is no CPU fallback: if no CUDA device is usable, calls that need one
 *     return SK_ECUDA.
 */
#ifndef COMPASS_B200_H
#define COMPASS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SK_API __attribute__((visibility("default")))
#else
#define SK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SK_OK = 0,
    SK_EINVAL = 1,       /* bad argument: arity/type, even d, non-power-of-two w */
    SK_EMISMATCH = 2,    /* seed / shape / edge mismatch on merge or estimate    */
    SK_EOVERFLOW = 3,    /* a counter or estimate bound would overflow; contraction unsupported    */
    SK_ENOMEM = 4,       /* allocation failure                                                       */
    SK_ECUDA = 5         /* CUDA runtime error / no device                                          */
} sk_status;

typedef struct sk_sketch sk_sketch;   /* opaque */

/* ---------------------------------------------------------------------------
 * Sketch descriptor.
 *   d            rows (independent basic estimators), odd, 1 <= d <= 63
 *                (PAPER.md:192 rows; median needs odd d).
 *   ndim         1: Fast-AGMS vector  sk[r][j]
 *                2: partitioned matrix M[r][i][j]
 *                3: partitioned tensor T[r][i][j][k]  ("a table with 3 joins
 *                   has a 3-D tensor as its sketch, with one dimension for every join
 *                   attribute")
 *   w[0..ndim)   buckets per dimension, powers of two in [2, 2^24]
 *                (PAPER.md:395 uses 1023; powers of two enable folding).
 *   master_seed  seed of the hash family (default 42).
 *   edge_id[q]   canonical join-edge id of dimension q: the two "alias.column"
 *                names sorted and joined by '|'.  Both sides of a
 *                join use the same id and therefore the same xi/h family
 *                (PAPER.md:148, 197); for ndim=2, strcmp(edge_id[0], edge_id[1]) < 0
 *                (dimension 0 = canonically first edge).
 * Hash family: x = key mod (2^61-1) after sign extension;
 *   xi_r(x) = +1 iff ((a3 x + a2) x + a1) x + a0 mod p is odd, else -1;
 *   h_r(x)  = ((b1 x + b0) mod p) mod w.
 * ------------------------------------------------------------------------- */
typedef struct {
    uint32_t d;
    uint32_t ndim;
    uint32_t w[3];
    uint64_t master_seed;
    const char *edge_id[3];
} sk_desc;

/* Counter layout: int64, row-major, [d][w0], [d][w0][w1] or [d][w0][w1][w2]; the
 * dimensions of a matrix or tensor are in canonical edge order (edge_id[0] < edge_id[1]
 * < edge_id[2]), else SK_EINVAL. */

/* Create a sketch on CUDA `device`.  counters_dev: caller-owned device buffer of
 * d*w0(*w1) int64 (must already be zeroed if a fresh sketch is wanted), or NULL
 * for a library-owned, zeroed buffer.  *out receives the handle. */
SK_API sk_status sketch_create(const sk_desc *desc, int device, int64_t *counters_dev, sk_sketch **out);

/* Destroy a handle (frees library-owned counters; never caller-owned ones).
 * Synchronises the device first.  NULL is a no-op. */
SK_API sk_status sketch_destroy(sk_sketch *sk);

/* Device pointer and number of int64 counters of a sketch. */
SK_API sk_status sketch_counters(const sk_sketch *sk, int64_t **counters_dev, uint64_t *n_counters);

/* Zero all counters (async on stream). */
SK_API sk_status sketch_zero(sk_sketch *sk, void *stream);

/* ---------------------------------------------------------------------------
 * sketch_update_filtered — the fused scan ("sketch building is
 * performed during the selection"; PAPER.md:99 one sketch per join attribute;
 * SPEC.md:288-296).  One pass over n_rows tuples of a columnar table:
 *   survive(i) = AND over preds of
 *       POINT : v == lo
 *       RANGE : lo <= v <= hi        (inclusive; use INT64_MIN / INT64_MAX for open ends)
 *       SUBSET: v in set[0..set_size)  (set is a HOST array, copied by the call;
 *                                       set_size == 0 means no value qualifies)
 *   with v = cols[pred.col][i] sign-extended to int64.  n_preds == 0 keeps all rows.
 *   For every surviving tuple and every target t, row r of t's sketch gets
 *       ndim 1: sk[r][h_r(k0)]              += xi_r(k0)
 *       ndim 2: M[r][h0_r(k0)][h1_r(k1)]     += xi0_r(k0) * xi1_r(k1)
 *       ndim 3: T[r][h0_r(k0)][h1_r(k1)][h2_r(k2)] += xi0_r(k0) xi1_r(k1) xi2_r(k2)
 *   with kq = cols[target.key_col[q]][i].
 *   *survivors_dev (device int64, may be NULL) += number of surviving tuples
 *   (the exact selection cardinality).
 * cols: device pointers, each n_rows elements of int32 or int64, 16-byte aligned
 *   recommended.  A key column of a table with predicates may also be pinned, mapped host
 *   memory (UVA): the scan reads only the survivors' key sectors in place over PCIe.  Counters are accumulated (+=), so calls over row shards add up
 *   (linearity).
 * Limits: n_cols <= 16, n_preds <= 8, n_targets <= 16, all targets on one device.
 * ------------------------------------------------------------------------- */
typedef enum { SK_INT32 = 0, SK_INT64 = 1 } sk_dtype;
typedef struct {
    const void *data;   /* device pointer */
    uint32_t dtype;     /* sk_dtype */
    uint64_t domain;    /* optional hint: key values lie in [0, domain); 0 = unknown.  With a
                           hint <= 2^22: int32 key columns (<= 2 keys, <= 2 predicates) take the
                           lookup-table path (one 16-byte table entry holds the (bucket, sign) of
                           every row of the key's hash family; matrices reuse it); otherwise the
                           1-D sketches of the column are built by histogram-then-sketch (one L2
                           atomic per surviving tuple, hashing once per distinct key).  Both are
                           exact by linearity; values outside the hinted domain
                           are still counted exactly (hashed directly).  A predicate column's
                           hint also sets the expected selectivity the scan is tuned for. */
} sk_column;

typedef enum { SK_PRED_POINT = 0, SK_PRED_RANGE = 1, SK_PRED_SUBSET = 2 } sk_pred_kind;
typedef struct {
    uint32_t col;        /* index into cols */
    uint32_t kind;       /* sk_pred_kind */
    int64_t lo, hi;      /* POINT uses lo; RANGE [lo, hi] */
    const int64_t *set;  /* SUBSET: host array (any order, duplicates allowed) */
    uint64_t set_size;
} sk_pred;

typedef struct {
    sk_sketch *sketch;
    uint32_t key_col[3]; /* key column per sketch dimension */
} sk_target;

SK_API sk_status sketch_update_filtered(const sk_column *cols, uint32_t n_cols, uint64_t n_rows,
                                 const sk_pred *preds, uint32_t n_preds,
                                 const sk_target *targets, uint32_t n_targets,
                                 int64_t *survivors_dev, void *stream);

/* dst += src elementwise (PAPER.md:86 mergeability).  Requires an
 * identical descriptor (d, ndim, w, master_seed, edge ids), else SK_EMISMATCH.
 * Cross-GPU merge: all-reduce (SUM, int64) the counter buffers with NCCL. */
SK_API sk_status sketch_merge(sk_sketch *dst, const sk_sketch *src, void *stream);

/* int32 wire format of the cross-GPU merge (SURVEY.md §8(e) lever i): the
 * all-reduce moves half the bytes when every partial and merged counter fits int32, which
 * holds whenever every table has < 2^31 rows (|counter| <= survivors <= rows).
 *   sketch_wire_pack:   wire_dev[i] = (int32) counters_dev[i], i < n; a value outside int32
 *                       sets *overflow_dev to 1 (device uint32, optional, never cleared).
 *   sketch_wire_unpack: counters_dev[i] = (int64) wire_dev[i], i < n.
 * Device buffers, caller-owned; asynchronous on `stream`; SK_EINVAL on NULL buffers with n > 0. */
SK_API sk_status sketch_wire_pack(const int64_t *counters_dev, int32_t *wire_dev, uint64_t n, unsigned int *overflow_dev,
                                  void *stream);
SK_API sk_status sketch_wire_unpack(const int32_t *wire_dev, int64_t *counters_dev, uint64_t n, void *stream);

/* ---------------------------------------------------------------------------
 * Cross-GPU merge over peer memory (SURVEY.md §8(f) 4, P2P variant of the fused flush +
 * all-reduce; "partition, sketch, merge").  Each rank owns a MERGED buffer with
 * the query's packed layout, allocated with sk_ipc_alloc and mapped into every other rank's
 * process with sk_ipc_open (handles exchanged by the caller, e.g. torch.distributed).  A push
 * adds this rank's partial slice into the same slice of every rank's merged buffer (own
 * included) with red.add over NVLink; once every rank's pushes have completed (caller: stream
 * synchronize + a host barrier), every merged buffer holds the sum of all partials — exact,
 * order-independent integer addition.  The merged buffers must be zeroed on every rank before
 * any rank pushes (caller: zero, synchronize, barrier).
 *   src:     this rank's partial slice (device, 16-byte aligned, n int64)
 *   dst:     host array of n_peers device pointers (1 <= n_peers <= 8): the slice in every
 *            rank's merged buffer as mapped in this process (16-byte aligned)
 * sketch_update_filtered_push: sketch_update_filtered, then the push of `src` — FUSED into the
 *   scan when the optimised kernel runs without a histogram epilogue: a cooperative launch
 *   whose CTAs, after a grid barrier that follows the last flush, push the slice (no separate
 *   kernel, no NCCL); otherwise (grid-stride kernel, histogram epilogue, or a refused
 *   cooperative launch) one k_peer_push launch after the scan.  `src` must cover the counters
 *   of every target (the table's slice of the partial buffer).
 * sketch_peer_push: the push alone (e.g. the survivor counts).
 * Errors: SK_EINVAL (NULL pointers, misalignment, n_peers out of range), SK_ECUDA. */
typedef struct {
    const int64_t *src;
    int64_t *const *dst;
    uint32_t n_peers;
    uint64_t n;
    /* owner_mode 1 (reduce-scatter over peer memory): the merged buffer of `total` elements is
     * split into n_peers contiguous ranges (range o starts at floor(total*o/n_peers) rounded
     * down to even); element i of src (merged-buffer index offset+i, offset even) is added
     * into its owner's buffer only, so each rank sends its partial once; after every rank's
     * pushes (caller barrier) sketch_peer_gather copies the other owners' ranges into this
     * rank's buffer (P2P reads).  owner_mode 0: added into every rank's buffer (one shot). */
    uint32_t owner_mode;
    uint32_t rank;      /* this rank (index into dst) */
    uint64_t offset;    /* owner_mode: element offset of src in the merged buffer */
    uint64_t total;     /* owner_mode: elements of the merged buffer */
} sk_peer_push;
SK_API sk_status sketch_update_filtered_push(const sk_column *cols, uint32_t n_cols, uint64_t n_rows,
                                             const sk_pred *preds, uint32_t n_preds,
                                             const sk_target *targets, uint32_t n_targets,
                                             int64_t *survivors_dev, const sk_peer_push *push, void *stream);
SK_API sk_status sketch_peer_push(const sk_peer_push *push, void *stream);
/* After an owner-mode merge: dst[rank][i] = dst[owner(i)][i] for every i < total owned by
 * another rank (dst = every rank's merged-buffer base as mapped here; src, n, offset unused). */
SK_API sk_status sketch_peer_gather(const sk_peer_push *push, void *stream);

/* CUDA IPC for the merged buffers.  sk_ipc_alloc: `bytes` of zeroed device memory on `device`
 * (library-owned until sk_ipc_free) and its SK_IPC_HANDLE_BYTES-byte handle.  sk_ipc_open:
 * map another process's buffer (never this process's own) on `device`; sk_ipc_close unmaps.
 * SK_EINVAL on NULL arguments, SK_ENOMEM, SK_ECUDA. */
#define SK_IPC_HANDLE_BYTES 64
SK_API sk_status sk_ipc_alloc(uint64_t bytes, int device, void **dev_ptr, unsigned char *handle);
SK_API sk_status sk_ipc_free(void *dev_ptr);
SK_API sk_status sk_ipc_open(const unsigned char *handle, int device, void **dev_ptr);
SK_API sk_status sk_ipc_close(void *dev_ptr);

/* ---------------------------------------------------------------------------
 * Join graph of one query: tables are vertices carrying their
 * exact post-selection cardinality; edge e joins tables edge_u[e] and edge_v[e]
 * and carries one 1-D sketch per side (vec_u[e] built on table edge_u[e]'s join
 * column, vec_v[e] on edge_v[e]'s), both with the edge's id and seed.  Optional
 * partitioned sketches: mat[m] is table mat_table[m]'s 2-D matrix over edges
 * (mat_e0[m], mat_e1[m]) (dimension 0 = mat_e0, the canonically first edge), or its 3-D
 * tensor (ndim 3; mat_e0/mat_e1 = its first two edges).  A table uses its
 * matrix or tensor in a sub-plan whose edges at that table are exactly the sketch's edges
 * (matched by edge id), else the min-abs merged view of its 1-D sketches.
 * All arrays are host arrays; sketches live on one device.  n_tables <= 64.
 * ------------------------------------------------------------------------- */
typedef struct {
    uint32_t n_tables;
    const int64_t *survivors;          /* [n_tables] */
    uint32_t n_edges;
    const uint32_t *edge_u, *edge_v;   /* [n_edges] */
    sk_sketch *const *vec_u;           /* [n_edges] */
    sk_sketch *const *vec_v;           /* [n_edges] */
    uint32_t n_mats;
    const uint32_t *mat_table;         /* [n_mats] */
    const uint32_t *mat_e0, *mat_e1;   /* [n_mats] */
    sk_sketch *const *mat;             /* [n_mats] */
} sk_graph;

/* ---------------------------------------------------------------------------
 * estimate_join — cardinality estimate of the connected sub-plan whose tables
 * are the set bits of vertex_mask:
 *   |C| = 1: the exact survivors of that table.
 *   |C| >= 2: per row r, E_r = sum over bucket assignments to every edge induced
 *     by C of the product of the tables' tensors, where a table contributes its
 *     1-D sketch (one incident edge in C), its matrix (if one is built over exactly
 *     its incident edges), or the min-abs merged view of its 1-D
 *     sketches in canonical edge order.  Vectors are folded to
 *     the narrowest width on each edge.
 *     Two-way: E_r = sum_j A[r][j] B[r][j].  Est = median_r E_r
 *     (PAPER.md:201), computed exactly (integer arithmetic), rounded once to fp64.
 * est: host double.  row_est: host double[d] or NULL (per-row E_r, rounded).
 * Supported: induced graphs with at most one independent cycle and tables with
 * at most 3 incident edges (SK_EOVERFLOW otherwise).  Synchronises `stream`.
 * ------------------------------------------------------------------------- */
SK_API sk_status estimate_join(const sk_graph *g, uint64_t vertex_mask, double *est, double *row_est, void *stream);

/* Same, but writes each row's exact E_r as a decimal string into
 * buf[r*stride .. r*stride+stride) (NUL-terminated); stride >= 160 recommended.
 * A singleton mask has no rows: its exact survivor count is written once, at buf[0]. */
SK_API sk_status estimate_join_exact(const sk_graph *g, uint64_t vertex_mask, char *buf, uint32_t stride, void *stream);

/* Batched estimates of n sub-plans: est[i] for masks[i]. */
SK_API sk_status estimate_subplans(const sk_graph *g, const uint64_t *masks, uint32_t n, double *est, void *stream);

/* ---------------------------------------------------------------------------
 * plan_greedy — greedy left-deep join order ("greedy", default in
 * the experiments PAPER.md:395):
 *   card(S) = survivors for |S| = 1, max(Est(S), 0) otherwise;
 *   start pair = edge (u, v) with least card, ties by (min index, max index);
 *   source = its endpoint with fewer survivors (ties: lower index);
 *   repeatedly append the neighbour v of C minimising card(C + v) (ties: lower
 *   index); cost = sum of card over all prefixes (Alg. 1 lines 14-15,
 *   PAPER.md:325-326).
 * order: host uint32[n_tables]; prefix_card: host double[n_tables]; cost: host.
 * Table index order must match the alias order used for ties.  Synchronises.
 * ------------------------------------------------------------------------- */
SK_API sk_status plan_greedy(const sk_graph *g, uint32_t *order, double *prefix_card, double *cost, void *stream);

/* ---------------------------------------------------------------------------
 * plan_enumerate — Algorithm 1 of the paper ("Fast-AGMS Sketch
 * Join Order Enumeration") with the search-space settings of PAPER.md:662:
 *   sources: all vertices in increasing f(v) = alpha*card(v)/max card +
 *     beta*deg(v)/max deg (line 7; card = exact survivors, deg = incident edges,
 *     parallel edges counted; ties: lower index);
 *   DFS Traversal(C, cost): cost += card(C) (lines 14-15); if cost > min_cost
 *     return (early pruning, line 17; skipped when cfg->no_prune); if |C| = |V|:
 *     keep C if cost < min_cost (strict, first found wins), p += 1, and stop the
 *     current source when p = max_plans (lines 19-26); else visit the
 *     neighbours v of C in increasing card(C + v) (ties: lower index, lines 29-35);
 *   card(S) = survivors for |S| = 1, max(Est(S), 0) otherwise;
 *     every estimate is computed once (cache; all connected sub-plans are estimated
 *     in one batch when there are at most 512 of them).
 *   mode SK_ENUM_GREEDY: plan_greedy's single-source rule (PAPER.md:662 greedy);
 *   SK_ENUM_FULL_GREEDY: max_plans = 1 from every source; SK_ENUM_LIMIT: max_plans =
 *   cfg->max_plans (paper default 10); SK_ENUM_EXHAUSTIVE: unbounded.
 * order/prefix_card: host arrays [n_tables] (the chosen plan and its per-prefix
 * cards); cost: host; stats: host or NULL.  Ties by index: table index order must
 * match the alias order.  SK_EINVAL on a NULL/ill-formed graph or config.
 * Synchronises `stream`.
 * ------------------------------------------------------------------------- */
typedef enum { SK_ENUM_GREEDY = 0, SK_ENUM_FULL_GREEDY = 1, SK_ENUM_LIMIT = 2, SK_ENUM_EXHAUSTIVE = 3 } sk_enum_mode;
typedef struct {
    double alpha, beta;     /* f(v) weights (paper default 0.5, 0.5) */
    uint32_t mode;          /* sk_enum_mode */
    uint32_t max_plans;     /* SK_ENUM_LIMIT: plans per source (>= 1) */
    uint32_t no_prune;      /* 1: disable early pruning (line 17); for checks */
} sk_enum_config;
typedef struct {
    uint64_t plans_completed;   /* complete plans reached (all sources) */
    uint64_t prunes;            /* branches cut by early pruning */
    uint64_t estimator_calls;   /* card() evaluations (cache hits included) */
    uint64_t distinct_estimates;/* sub-plans estimated (cache size) */
} sk_enum_stats;
SK_API sk_status plan_enumerate(const sk_graph *g, const sk_enum_config *cfg, uint32_t *order, double *prefix_card,
                                double *cost, sk_enum_stats *stats, void *stream);

/* ---------------------------------------------------------------------------
 * exact_join_size — the exact cardinality |R_1 join ... join R_k| of a connected sub-plan
 * (cycles and parallel edges included), for the accuracy evaluation of the estimates
 * (accuracy ratio est/true over "all the enumerated sub-plans"; normalised L1
 * distance of orderings).
 * Frequency-vector message passing on the device: a leaf table sends f(k) = number of its
 * surviving tuples with join key k; an inner table sends, for each key of its parent edge,
 * the sum over its surviving tuples of the product of its children's messages at the
 * tuple's keys; the root sums that product over its surviving tuples.  Exact: every pass is
 * modulo K primes < 2^26 (K from the bound prod_t n_rows_t) and the count is reconstructed
 * by CRT on the host.  Cycles: an induced edge whose two columns are already equal through
 * other edges (transitivity of equality, e.g. a triangle on one key column per table) is
 * implied and dropped; a remaining cycle is conditioned on one of its edges, summing the
 * acyclic count with both endpoints' columns fixed to k over every k of that edge's key
 * domain (at most 65536 conditioned keys per call).
 *   tables[t]: n_rows, device columns, predicates exactly as sketch_update_filtered
 *     (survive(i) = AND of the predicates).
 *   edge e joins table edge_u[e] column col_u[e] with table edge_v[e] column col_v[e];
 *     every join key of a surviving tuple must lie in [key_lo[e], key_lo[e] + key_domain[e])
 *     (SK_EINVAL otherwise; key_domain[e] <= 2^31).
 *   vertex_mask: the sub-plan (>= 1 table; a single table gives its survivor count).
 * dec: host buffer receiving the count in decimal (NUL-terminated, dec_len >= 2), or NULL;
 * approx: host double (the count rounded to nearest), or NULL.
 * SK_EOVERFLOW for a cycle whose conditioning exceeds 65536 keys, for tables with more than
 * 4 tree edges, or more than 8 predicates after conditioning.  Synchronises `stream`.
 * ------------------------------------------------------------------------- */
typedef struct {
    uint64_t n_rows;
    const sk_column *cols;
    uint32_t n_cols;
    const sk_pred *preds;
    uint32_t n_preds;
} sk_table_data;
typedef struct {
    uint32_t n_tables;
    const sk_table_data *tables;   /* [n_tables] */
    uint32_t n_edges;
    const uint32_t *edge_u, *edge_v, *col_u, *col_v;   /* [n_edges] */
    const int64_t *key_lo;         /* [n_edges] */
    const uint64_t *key_domain;    /* [n_edges] */
} sk_join_data;
SK_API sk_status exact_join_size(const sk_join_data *jd, uint64_t vertex_mask, char *dec, uint32_t dec_len,
                                 double *approx, void *stream);

/* Thread-local description of the last error (never NULL). */
SK_API const char *sk_last_error(void);

/* Number of CUDA kernels this library has launched since it was loaded
 * (diagnostic; lets a caller count the library's launches in a timed region). */
SK_API uint64_t sk_kernel_launches(void);

/* Library build / device information, e.g. "compass_b200 sm_100a". */
SK_API const char *sk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* COMPASS_B200_H */
