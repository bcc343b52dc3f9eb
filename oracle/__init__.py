"""CPU oracle for the COMPASS Fast-AGMS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2102_02440_b200``) never imports it and shares no code with it.

The arithmetic lives in ``compass_oracle.c`` (plain C, built to ``liboracle.so``);
this module marshals numpy arrays and writes out, in plain Python, the two pieces
of logic that are bookkeeping over at most ~10 tables:

* ``subplan_tensors`` — which tensor each table contributes to a sub-plan
  ("separate sketches are required for every
  join", PAPER.md:234-240 merging, PAPER.md:225 same-bucket-count constraint →
  fold).
* ``plan_greedy`` — the greedy left-deep enumerator (SURVEY.md
  §8(c) O10; Alg. 1 cost lines 14-15).

Parity status per function: see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from itertools import combinations

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "compass_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

POINT, RANGE, SUBSET = 0, 1, 2
K_VEC, K_MAT, K_MERGED, K_TEN3 = 0, 1, 2, 3   # K_TEN3: 3-D partitioned tensor
INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1


def build_oracle(force: bool = False) -> str:
    """Compile compass_oracle.c with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_LIB)
        u64, i64, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
        vp, cp = ctypes.c_void_p, ctypes.c_char_p
        L.or_splitmix64.restype = u64; L.or_splitmix64.argtypes = [u64]
        L.or_fnv1a64.restype = u64; L.or_fnv1a64.argtypes = [cp]
        L.or_coef.restype = u64; L.or_coef.argtypes = [u64, cp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.or_canon.restype = u64; L.or_canon.argtypes = [i64]
        L.or_xi.restype = i32; L.or_xi.argtypes = [u64, cp, ctypes.c_uint32, i64]
        L.or_bucket.restype = u64; L.or_bucket.argtypes = [u64, cp, ctypes.c_uint32, i64, u64]
        L.or_filter.restype = i64
        L.or_filter.argtypes = [i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp]
        L.or_build.restype = i32
        L.or_build.argtypes = [i64, vp, vp, i32, vp, i32, i32, i32, vp, cp, cp, u64, vp]
        L.or_build_nd.restype = i32
        L.or_build_nd.argtypes = [i64, vp, i32, vp, vp, i32, vp, vp, u64, vp]
        L.or_contract_row.restype = i32
        L.or_contract_row.argtypes = [i32, vp, vp, vp, vp, i32, vp, cp, i32, vp]
        L.or_contract_brute_row.restype = i32
        L.or_contract_brute_row.argtypes = [i32, vp, vp, vp, vp, i32, vp, cp, i32, vp]
        L.or_two_way_row.restype = i32
        L.or_two_way_row.argtypes = [i64, vp, vp, cp, i32, vp]
        L.or_bn_selftest_mul_add.restype = i32
        L.or_bn_selftest_mul_add.argtypes = [i32, vp, vp, cp, i32]
        L.or_bn_selftest_to_double.restype = ctypes.c_double
        L.or_bn_selftest_to_double.argtypes = [i32, vp]
        L.or_dec_to_double.restype = ctypes.c_double
        L.or_dec_to_double.argtypes = [cp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------------
# H1-H4 (hash family / seeds)
# --------------------------------------------------------------------------

def coef(master: int, edge_id: str, row: int, role: int, idx: int) -> int:
    return lib().or_coef(master, edge_id.encode(), row, role, idx)


def canon(key: int) -> int:
    return lib().or_canon(key)


def xi(master: int, edge_id: str, row: int, key: int) -> int:
    return lib().or_xi(master, edge_id.encode(), row, key)


def bucket(master: int, edge_id: str, row: int, key: int, w: int) -> int:
    return lib().or_bucket(master, edge_id.encode(), row, key, w)


# --------------------------------------------------------------------------
# O1 filter / O2-O3 build / O4 merge / O5 fold
# --------------------------------------------------------------------------

def filter_mask(columns: dict, preds: list) -> tuple[np.ndarray, int]:
    """preds: list of (col_name, kind, lo, hi, set_values_or_None).  Conjunction (O1)."""
    preds = [tuple(p) + (None,) * (5 - len(p)) for p in preds]
    names = list(columns)
    n = len(columns[names[0]]) if names else 0
    cols = [np.ascontiguousarray(columns[k]) for k in names]
    for c in cols:
        assert c.dtype in (np.int32, np.int64)
    colp = (ctypes.c_void_p * max(1, len(cols)))(*[_ptr(c) for c in cols])
    is64 = np.array([1 if c.dtype == np.int64 else 0 for c in cols], dtype=np.int32)
    npred = len(preds)
    pcol = np.array([names.index(p[0]) for p in preds] or [0], dtype=np.int32)
    pkind = np.array([p[1] for p in preds] or [0], dtype=np.int32)
    plo = np.array([p[2] for p in preds] or [0], dtype=np.int64)
    phi = np.array([p[3] for p in preds] or [0], dtype=np.int64)
    sets = [np.ascontiguousarray(np.asarray(p[4] if p[4] is not None else [], dtype=np.int64)) for p in preds]
    psetp = (ctypes.c_void_p * max(1, npred))(*[_ptr(s) if len(s) else 0 for s in sets])
    psetn = np.array([len(s) for s in sets] or [0], dtype=np.int64)
    mask = np.zeros(n, dtype=np.uint8)
    cnt = lib().or_filter(n, ctypes.cast(colp, ctypes.c_void_p), _ptr(is64), npred, _ptr(pcol), _ptr(pkind),
                          _ptr(plo), _ptr(phi), ctypes.cast(psetp, ctypes.c_void_p), _ptr(psetn), _ptr(mask))
    return mask, int(cnt)


def build(keys: list, mask, d: int, w: list, edge_ids: list, master: int = 42, out=None) -> np.ndarray:
    """Fast-AGMS sketch (ndim = len(keys) = 1), partitioned matrix (ndim 2), O2/O3, or 3-D
    partitioned tensor (ndim 3), dims in the given (canonical) edge order."""
    ndim = len(keys)
    assert ndim in (1, 2, 3) and len(w) == ndim and len(edge_ids) == ndim
    n = len(keys[0])
    shape = (d, *w)
    if out is None:
        out = np.zeros(shape, dtype=np.int64)
    assert out.shape == shape and out.dtype == np.int64 and out.flags.c_contiguous
    m = np.ascontiguousarray(mask, dtype=np.uint8) if mask is not None else None
    wa = np.array(w, dtype=np.int64)
    if ndim == 3:
        ks = [np.ascontiguousarray(k) for k in keys]
        kp = (ctypes.c_void_p * 3)(*[_ptr(k) for k in ks])
        is64 = np.array([int(k.dtype == np.int64) for k in ks], dtype=np.int32)
        eb = [e.encode() for e in edge_ids]
        ep = (ctypes.c_char_p * 3)(*eb)
        rc = lib().or_build_nd(n, _ptr(m) if m is not None else 0, 3, ctypes.cast(kp, ctypes.c_void_p), _ptr(is64), d,
                               _ptr(wa), ctypes.cast(ep, ctypes.c_void_p), master, _ptr(out))
        assert rc == 0
        return out
    k0 = np.ascontiguousarray(keys[0])
    k1 = np.ascontiguousarray(keys[1]) if ndim == 2 else k0
    rc = lib().or_build(n, _ptr(m) if m is not None else 0,
                        _ptr(k0), int(k0.dtype == np.int64), _ptr(k1), int(k1.dtype == np.int64),
                        d, ndim, _ptr(wa), edge_ids[0].encode(), edge_ids[-1].encode(), master, _ptr(out))
    assert rc == 0
    return out


def fold(v: np.ndarray, w_new: int, axis: int = -1) -> np.ndarray:
    """O5: v'[j] = sum_t v[j + t*w']."""
    v = np.asarray(v)
    axis = axis % v.ndim
    w = v.shape[axis]
    assert w % w_new == 0
    shp = v.shape[:axis] + (w // w_new, w_new) + v.shape[axis + 1:]
    return v.reshape(shp).sum(axis=axis)


# --------------------------------------------------------------------------
# O6 / O7 estimates
# --------------------------------------------------------------------------

def _call_contract(fn, tensors, widths):
    """tensors: list of (kind, legs(list of edge idx), [arrays...]) for one row."""
    T = len(tensors)
    kind = np.array([t[0] for t in tensors], dtype=np.int32)
    nlegs = np.array([len(t[1]) for t in tensors], dtype=np.int32)
    legs = np.full(3 * T, -1, dtype=np.int32)
    keep = []
    ptrs = (ctypes.c_void_p * (3 * T))()
    for i, (k, lg, arrs) in enumerate(tensors):
        for q, e in enumerate(lg):
            legs[3 * i + q] = e
        for q, a in enumerate(arrs):
            a = np.ascontiguousarray(a, dtype=np.int64)
            keep.append(a)
            ptrs[3 * i + q] = _ptr(a)
    wa = np.array(widths, dtype=np.int64)
    buf = ctypes.create_string_buffer(256)
    dbl = ctypes.c_double(0.0)
    rc = fn(T, _ptr(kind), _ptr(nlegs), _ptr(legs), ctypes.cast(ptrs, ctypes.c_void_p), len(widths), _ptr(wa),
            buf, 256, ctypes.addressof(dbl))
    if rc != 0:
        raise RuntimeError(f"oracle contraction failed rc={rc}")
    return int(buf.value.decode())


def contract_row(tensors, widths, brute: bool = False) -> int:
    L = lib()
    return _call_contract(L.or_contract_brute_row if brute else L.or_contract_row, tensors, widths)


def two_way_row(a: np.ndarray, b: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.int64)
    assert a.shape == b.shape
    buf = ctypes.create_string_buffer(256)
    rc = lib().or_two_way_row(len(a), _ptr(a), _ptr(b), buf, 256, 0)
    assert rc == 0
    return int(buf.value.decode())


def median_odd(vals):
    """Median of an odd number of exact values: element (d-1)/2 of the ascending sort
    (even d rejected, reading R4)."""
    assert len(vals) % 2 == 1
    return sorted(vals)[(len(vals) - 1) // 2]


class Graph:
    """Join graph with its built sketches (SURVEY.md §8(b) sk_graph, oracle side).

    tables: {alias: survivors}; edges: list of (edge_id, u, v);
    vec: {(alias, edge_id): int64[d][w]}; mat: {(alias, (e_lo, e_hi)): int64[d][w_lo][w_hi]} and
    3-D tensors {(alias, (e_0, e_1, e_2)): int64[d][w_0][w_1][w_2]}, edges canonical.
    """

    def __init__(self, tables, edges, vec, mat=None):
        self.tables = dict(tables)
        self.edges = sorted(edges)  # canonical order = edge-id string order (H2)
        self.vec = dict(vec)
        self.mat = dict(mat or {})
        self.d = next(iter(self.vec.values())).shape[0]

    def induced(self, subset):
        s = set(subset)
        return [e for e in self.edges if e[1] in s and e[2] in s]


def subplan_tensors(g: Graph, subset):
    """Per SURVEY.md O7: which tensor each table contributes, and the common
    width per edge (fold to the narrowest, PAPER.md:225 same bucket count).
    Returns (tables, edge_list, widths, per_row_fn)."""
    E = g.induced(subset)
    eidx = {e[0]: i for i, e in enumerate(E)}
    specs = []
    for t in sorted(subset):
        inc = [e[0] for e in E if t in (e[1], e[2])]  # canonical order
        if len(inc) == 1:
            specs.append((t, K_VEC, inc, [g.vec[(t, inc[0])]]))
        elif len(inc) == 2 and (t, (inc[0], inc[1])) in g.mat:
            specs.append((t, K_MAT, inc, [g.mat[(t, (inc[0], inc[1]))]]))
        elif len(inc) == 3 and (t, tuple(inc)) in g.mat:          # PAPER.md:225 3-D tensor
            specs.append((t, K_TEN3, inc, [g.mat[(t, tuple(inc))]]))
        else:
            specs.append((t, K_MERGED, inc, [g.vec[(t, e)] for e in inc]))
    # widths: narrowest native width seen on each edge
    widths = [None] * len(E)
    for t, kind, inc, arrs in specs:
        for q, e in enumerate(inc):
            if kind in (K_MAT, K_TEN3):
                wn = arrs[0].shape[1 + q]
            elif kind == K_VEC:
                wn = arrs[0].shape[1]
            else:
                wn = arrs[q].shape[1]
            i = eidx[e]
            widths[i] = wn if widths[i] is None else min(widths[i], wn)
    # fold every leg to its edge width (O5)
    folded = []
    for t, kind, inc, arrs in specs:
        if kind in (K_MAT, K_TEN3):
            m = arrs[0]
            for q, e in enumerate(inc):
                m = fold(m, widths[eidx[e]], axis=1 + q)
            folded.append((kind, [eidx[e] for e in inc], [m]))
        elif kind == K_VEC:
            folded.append((kind, [eidx[inc[0]]], [fold(arrs[0], widths[eidx[inc[0]]], axis=1)]))
        else:
            folded.append((kind, [eidx[e] for e in inc],
                           [fold(a, widths[eidx[e]], axis=1) for a, e in zip(arrs, inc)]))
    return folded, widths


def estimate_rows(g: Graph, subset, brute: bool = False, rows=None):
    """Exact per-row E_r (Python ints) for a connected sub-plan with >= 2 tables."""
    folded, widths = subplan_tensors(g, subset)
    out = []
    for r in (range(g.d) if rows is None else rows):
        tens = []
        for kind, legs, arrs in folded:
            if kind in (K_MAT, K_TEN3):
                tens.append((kind, legs, [arrs[0][r].reshape(-1)]))
            else:
                tens.append((kind, legs, [a[r] for a in arrs]))
        out.append(contract_row(tens, widths, brute=brute))
    return out


def estimate(g: Graph, subset, brute: bool = False):
    """Est = median over rows (signed), as fp64 (correctly rounded once)."""
    subset = tuple(sorted(subset))
    if len(subset) == 1:
        return float(g.tables[subset[0]]), None
    rows = estimate_rows(g, subset, brute=brute)
    return float(median_odd(rows)), rows


def connected(g: Graph, subset) -> bool:
    s = set(subset)
    if not s:
        return False
    start = next(iter(s))
    seen = {start}
    stack = [start]
    while stack:
        t = stack.pop()
        for _, u, v in g.edges:
            for a, b in ((u, v), (v, u)):
                if a == t and b in s and b not in seen:
                    seen.add(b)
                    stack.append(b)
    return seen == s


def connected_subplans(g: Graph, min_size: int = 2):
    names = sorted(g.tables)
    out = []
    for k in range(min_size, len(names) + 1):
        for c in combinations(names, k):
            if connected(g, c):
                out.append(c)
    return out


def plan_greedy(g: Graph, est_fn=None):
    """Greedy left-deep enumeration.

    card(S) = survivors for |S| = 1, max(Est, 0) otherwise.
    Returns (order, prefix_cards, cost)."""
    cache = {}

    def card(S):
        S = tuple(sorted(S))
        if S not in cache:
            if len(S) == 1:
                cache[S] = float(g.tables[S[0]])
            else:
                e = est_fn(S) if est_fn else estimate(g, S)[0]
                cache[S] = max(float(e), 0.0)
        return cache[S]

    names = sorted(g.tables)
    if len(names) == 1:
        c = card(names)
        return names, [c], c
    pairs = sorted({tuple(sorted((u, v))) for _, u, v in g.edges})
    best = min(pairs, key=lambda p: (card(p), p))
    source = min(best, key=lambda a: (g.tables[a], a))
    C = [source]
    prefix = [card(C)]
    cost = prefix[0]
    while len(C) < len(names):
        cand = sorted({b for _, u, v in g.edges for a, b in ((u, v), (v, u)) if a in C and b not in C})
        v = min(cand, key=lambda x: (card(C + [x]), x))
        C.append(v)
        c = card(C)
        prefix.append(c)
        cost += c
    return C, prefix, cost


def plan_enumerate(g: Graph, mode="limit", max_plans=10, alpha=0.5, beta=0.5, prune=True, est_fn=None,
                   card_fn=None):
    """Algorithm 1 of the paper, literally, with the search-space
    settings of PAPER.md:662 (greedy | full-greedy | limit | exhaustive).

    card(S) = survivors for |S| = 1, max(Est, 0) otherwise;
    card_fn(S) overrides card entirely (tests: any cardinality function).
    Sources in increasing f(v) = alpha*card(v)/max card + beta*deg(v)/max deg (line 7),
    ties by alias; DFS Traversal adds card(C) to cost (lines 14-15), returns when
    cost > min_cost (line 17, unless prune=False), records a complete plan if
    cost < min_cost (lines 20-23), counts it in p and stops the current source when
    p = max_plans (lines 24-25, per source: p is reset at line 9), and
    visits the neighbours of C in increasing card(C + v), ties by alias (lines 29-35).
    Returns (order, prefix_cards, cost, stats)."""
    if mode == "greedy":
        order, pre, cost = plan_greedy(g, est_fn)
        return order, pre, cost, {"plans_completed": 1}
    cache = {}

    def card(S):
        key = tuple(sorted(S))
        if key not in cache:
            if card_fn is not None:
                cache[key] = float(card_fn(key))
            elif len(key) == 1:
                cache[key] = float(g.tables[key[0]])
            else:
                e = est_fn(key) if est_fn else estimate(g, key)[0]
                cache[key] = max(float(e), 0.0)
        return cache[key]

    names = sorted(g.tables)
    adj = {a: set() for a in names}
    deg = {a: 0 for a in names}
    for _, u, v in g.edges:
        adj[u].add(v)
        adj[v].add(u)
        deg[u] += 1
        deg[v] += 1
    maxc = max(float(g.tables[a]) for a in names)
    maxd = max(deg.values())

    def f(v):
        return (alpha * float(g.tables[v]) / maxc if maxc > 0 else 0.0) + (beta * deg[v] / maxd if maxd > 0 else 0.0)

    S = sorted(names, key=lambda v: (f(v), v))
    limit = {"full-greedy": 1, "limit": max_plans, "exhaustive": None}[mode]
    st = {"min_cost": float("inf"), "opt": None, "p": 0, "abort": False,
          "plans_completed": 0, "prunes": 0}

    def dfs(C, cost):
        if st["abort"]:
            return
        cost = cost + card(C)                                   # lines 14-15
        if prune and cost > st["min_cost"]:                     # line 17
            st["prunes"] += 1
            return
        if len(C) == len(names):                                # lines 19-26
            if cost < st["min_cost"]:
                st["min_cost"], st["opt"] = cost, list(C)
            st["plans_completed"] += 1
            st["p"] += 1
            if limit is not None and st["p"] == limit:
                st["abort"] = True
            return
        L = sorted({b for a in C for b in adj[a]} - set(C))     # line 29
        e = {v: card(C + [v]) for v in L}                       # lines 30-32
        for v in sorted(L, key=lambda x: (e[x], x)):            # lines 33-35
            if st["abort"]:
                return
            dfs(C + [v], cost)

    for v in S:                                                 # lines 8-11
        st["p"], st["abort"] = 0, False
        dfs([v], 0.0)
    order = st["opt"]
    pre = [card(order[:i + 1]) for i in range(len(order))]
    return order, pre, st["min_cost"], {"plans_completed": st["plans_completed"], "prunes": st["prunes"]}


def leftdeep_costs_bruteforce(names, edges, card_fn):
    """Every valid left-deep order (each prefix connected, no cross products) with its
    cost sum_i card(prefix_i) — the exhaustive search space of PAPER.md:662."""
    from itertools import permutations
    adj = {a: set() for a in names}
    for _, u, v in edges:
        adj[u].add(v)
        adj[v].add(u)
    out = {}
    for perm in permutations(names):
        ok = all(any(p in adj[perm[i]] for p in perm[:i]) for i in range(1, len(perm)))
        if ok:
            out[perm] = sum(float(card_fn(tuple(sorted(perm[:i + 1])))) for i in range(len(perm)))
    return out


def exact_join_size(tables, edges, subset):
    """Exact |join| of an acyclic connected sub-plan (the truth of the
    accuracy ratio).  tables: {alias: (columns dict, preds)}; edges: list of
    (u, v, col_u, col_v); subset: aliases.  Message passing over the join tree with Python
    integers: a table sends, per key of its parent edge, the sum over its surviving tuples of
    the product of its children's messages at the tuple's keys.  Pinned by
    exact_join_size_bruteforce."""
    S = sorted(set(subset))
    E = [e for e in edges if e[0] in S and e[1] in S]
    if len(E) != len(S) - 1:
        raise ValueError("cyclic or disconnected sub-plan")
    masks = {t: filter_mask(tables[t][0], tables[t][1])[0] for t in S}
    root = S[0]

    def send(t, parent_edge):
        cols = tables[t][0]
        rows = np.nonzero(masks[t])[0]
        child = []
        for e in E:
            if e is parent_edge or t not in (e[0], e[1]):
                continue
            c, col = (e[1], e[2]) if e[0] == t else (e[0], e[3])
            child.append((col, send(c, e)))
        out = {}
        pcol = None if parent_edge is None else (parent_edge[2] if parent_edge[0] == t else parent_edge[3])
        total = 0
        for i in rows:
            v = 1
            for col, m in child:
                v *= m.get(int(cols[col][i]), 0)
                if v == 0:
                    break
            if pcol is None:
                total += v
            elif v:
                k = int(cols[pcol][i])
                out[k] = out.get(k, 0) + v
        return total if pcol is None else out
    return send(root, None)


def exact_join_size_any(tables, edges, subset) -> int:
    """Exact |join| of any connected sub-plan, cycles and parallel edges included (SURVEY.md
    §8(f) 2; PAPER.md:261 needs the truth of "all the enumerated sub-plans", and the paper's
    running example has a triangle).  A hash join with multiplicities: tables
    are joined one at a time (each new table adjacent to the joined set); the partial result
    is a map from the values of the joined tables' columns that still have edges to unjoined
    tables to the number of partial tuple combinations carrying them; a new table's surviving
    row extends exactly the entries whose values agree with it on EVERY edge between the new
    table and the joined set (an edge closing a cycle is one more equality checked).  Plain
    Python integers.  Pinned by exact_join_size_bruteforce on tiny cyclic graphs."""
    S = sorted(set(subset))
    E = [e for e in edges if e[0] in S and e[1] in S]
    masks = {t: filter_mask(tables[t][0], tables[t][1])[0] for t in S}
    order = [S[0]]
    while len(order) < len(S):
        nxt = [t for t in S if t not in order and any((u in order and v == t) or (v in order and u == t)
                                                     for u, v, _, _ in E)]
        if not nxt:
            raise ValueError("disconnected sub-plan")
        order.append(nxt[0])

    def open_cols(joined):
        """(table, col) of joined tables with an edge to a table not joined yet (sorted)."""
        out = set()
        for u, v, cu, cv in E:
            if u in joined and v not in joined:
                out.add((u, cu))
            if v in joined and u not in joined:
                out.add((v, cv))
        return sorted(out)

    joined = {order[0]}
    t0 = order[0]
    cols0 = tables[t0][0]
    oc = open_cols(joined)
    state = {}
    for i in np.nonzero(masks[t0])[0]:
        key = tuple(int(tables[t][0][c][i]) for t, c in oc)
        state[key] = state.get(key, 0) + 1
    for t in order[1:]:
        cols = tables[t][0]
        # edges between t and the joined set: (open-column position, column of t)
        links = []
        for u, v, cu, cv in E:
            if u == t and v in joined:
                links.append((oc.index((v, cv)), cu))
            elif v == t and u in joined:
                links.append((oc.index((u, cu)), cv))
        joined.add(t)
        oc_new = open_cols(joined)
        idx = {}   # state entries by the values the new table must match
        for key, cnt in state.items():
            idx.setdefault(tuple(key[p] for p, _ in links), []).append((key, cnt))
        new = {}
        for i in np.nonzero(masks[t])[0]:
            want = tuple(int(cols[c][i]) for _, c in links)
            for key, cnt in idx.get(want, ()):
                full = {tc: key[j] for j, tc in enumerate(oc)}
                for tt, c in oc_new:
                    if tt == t:
                        full[(t, c)] = int(cols[c][i])
                nk = tuple(full[tc] for tc in oc_new)
                new[nk] = new.get(nk, 0) + cnt
        state, oc = new, oc_new
    return sum(state.values())


def exact_join_size_bruteforce(tables, edges, subset) -> int:
    """The literal definition (tiny inputs only): the number of combinations of one surviving
    tuple per table that agree on every induced join edge."""
    from itertools import product
    S = sorted(set(subset))
    E = [e for e in edges if e[0] in S and e[1] in S]
    rows = {t: np.nonzero(filter_mask(tables[t][0], tables[t][1])[0])[0].tolist() for t in S}
    n = 0
    for combo in product(*[rows[t] for t in S]):
        pick = dict(zip(S, combo))
        if all(int(tables[u][0][cu][pick[u]]) == int(tables[v][0][cv][pick[v]]) for u, v, cu, cv in E):
            n += 1
    return n


def accuracy_report(estimates: dict, truths: dict):
    """PAPER.md:261 accuracy ratio est/true per sub-plan, and PAPER.md:294 normalised L1
    distance per sub-plan size (permutation_l1 / number of sub-plans of that size).
    estimates, truths: {sub-plan (tuple of aliases): value}.  Returns {size: (ratios, l1)}."""
    out = {}
    for size in sorted({len(s) for s in truths}):
        keys = sorted(s for s in truths if len(s) == size)
        ratios = [float(estimates[s]) / float(truths[s]) if truths[s] else float("inf") for s in keys]
        l1 = permutation_l1([estimates[s] for s in keys], [truths[s] for s in keys]) / len(keys)
        out[size] = (ratios, l1)
    return out


def permutation_l1(estimates, truths) -> int:
    """Normalised-L1 numerator: sum_i |S_i - C_i|, ranks by ascending
    value, ties by stable original index."""
    n = len(truths)
    order_t = sorted(range(n), key=lambda i: (truths[i], i))
    order_e = sorted(range(n), key=lambda i: (estimates[i], i))
    rank_t = {i: r for r, i in enumerate(order_t)}
    rank_e = {i: r for r, i in enumerate(order_e)}
    return sum(abs(rank_e[i] - rank_t[i]) for i in range(n))


def merge_entry(values):
    """Min-abs merge of bucket values, left fold."""
    acc = values[0]
    for v in values[1:]:
        if not (abs(acc) <= abs(v)):
            acc = v
    return acc
