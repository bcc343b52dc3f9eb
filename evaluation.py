"""Accuracy evaluation workload of the sketch estimates — evaluation
tooling beside the hot path, not part of it (it is not in the product package).

The truth of every connected sub-plan (cycles included) comes from ``exact_join_size``
(frequency-vector message passing in the library's CUDA kernels, exact by CRT; implied cycle
edges dropped, genuine cycles conditioned on one edge).  The two measures of the paper:
  * accuracy ratio = estimate / true cardinality per sub-plan;
  * normalised L1 distance per sub-plan size: sort the sub-plans of one size by true
    cardinality (order C) and by estimate (order S), sum |S_i - C_i| over the positions and
    divide by the number of sub-plans.
Host arithmetic only (no part of the hot path runs here).
"""
from __future__ import annotations

from itertools import combinations

from paper_2102_02440_b200 import SK_EOVERFLOW, SkError, exact_join_size


def join_data(ws, data: dict, preds: dict):
    """(tables, edges, names) for exact_join_size from a workload: tables in alias order, one
    edge per workload join edge with the join columns and the key domain of the generator."""
    names = sorted(t.name for t in ws.tables)
    tables, colpos = [], {}
    for n in names:
        t = ws.table(n)
        cols = [c.name for c in t.cols]
        colpos[n] = {c: i for i, c in enumerate(cols)}
        pr = []
        for p in preds[n]:
            c, kind, lo, hi, st = p
            pr.append((cols.index(c), kind, lo, hi, st))
        tables.append(([data[n][c] for c in cols], pr))
    keycol = {}
    for s in ws.sketches:
        if len(s.edge_ids) == 1:
            keycol[(s.table, s.edge_ids[0])] = s.key_cols[0]
    edges = []
    for eid, u, v in ws.edges:
        cu, cv = keycol[(u, eid)], keycol[(v, eid)]
        dom = max(ws.table(u).col(cu).domain, ws.table(v).col(cv).domain)
        edges.append((names.index(u), names.index(v), colpos[u][cu], colpos[v][cv], 0, dom))
    return tables, edges, names


def acyclic_connected_subplans(names, edges, min_size=2):
    """Vertex sets whose induced join graph is a tree (acyclic and connected)."""
    out = []
    for k in range(min_size, len(names) + 1):
        for sub in combinations(range(len(names)), k):
            s = set(sub)
            ind = [(u, v) for u, v, *_ in edges if u in s and v in s]
            if len(ind) != k - 1:
                continue
            seen, st = {sub[0]}, [sub[0]]
            while st:
                x = st.pop()
                for u, v in ind:
                    y = v if u == x else (u if v == x else None)
                    if y is not None and y not in seen:
                        seen.add(y)
                        st.append(y)
            if seen == s:
                out.append(tuple(names[i] for i in sub))
    return out


def connected_subplans(names, edges, min_size=2):
    """Every vertex set whose induced join graph is connected (cycles included)."""
    out = []
    for k in range(min_size, len(names) + 1):
        for sub in combinations(range(len(names)), k):
            s = set(sub)
            ind = [(u, v) for u, v, *_ in edges if u in s and v in s]
            seen, st = {sub[0]}, [sub[0]]
            while st:
                x = st.pop()
                for u, v in ind:
                    y = v if u == x else (u if v == x else None)
                    if y is not None and y not in seen:
                        seen.add(y)
                        st.append(y)
            if seen == s:
                out.append(tuple(names[i] for i in sub))
    return out


def exact_counts(tables, edges, names, subsets, stream=None) -> dict:
    """{sub-plan: exact count}; None where the library declines (a genuine cycle over a key
    domain too large to condition, SK_EOVERFLOW)."""
    out = {}
    for s in subsets:
        try:
            out[s] = exact_join_size(tables, edges, sum(1 << names.index(t) for t in s), stream)
        except SkError as ex:
            if ex.status != SK_EOVERFLOW:
                raise
            out[s] = None
    return out


def l1_distance(estimates, truths) -> int:
    """sum_i |S_i - C_i|: positions in the estimate order vs the true order,
    ties broken by the original index."""
    n = len(truths)
    pos_t = {i: r for r, i in enumerate(sorted(range(n), key=lambda i: (truths[i], i)))}
    pos_e = {i: r for r, i in enumerate(sorted(range(n), key=lambda i: (estimates[i], i)))}
    return sum(abs(pos_e[i] - pos_t[i]) for i in range(n))


def report(estimates: dict, truths: dict) -> dict:
    """{size: (accuracy ratios in sub-plan order, normalised L1 distance)}."""
    out = {}
    truths = {s: v for s, v in truths.items() if v is not None}
    for size in sorted({len(s) for s in truths}):
        keys = sorted(s for s in truths if len(s) == size)
        ratios = [float(estimates[s]) / float(truths[s]) if truths[s] else float("inf") for s in keys]
        out[size] = (ratios, l1_distance([estimates[s] for s in keys], [truths[s] for s in keys]) / len(keys))
    return out
