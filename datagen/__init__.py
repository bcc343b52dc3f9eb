"""Seeded synthetic inputs for the COMPASS hot path (configs C1-C5 of BASELINE.json).

This module holds NO arithmetic of the method (no hashing, filtering, sketching
or estimation).  It only describes workloads and generates their columns with a
counter-based generator, so that the same bytes can feed both the CUDA path and
the CPU oracle, and so that any row shard is a slice of the 1-GPU table:

    value = f(data_seed, table, column, global_row)

The generator is written with torch int64/float64 element-wise ops (identical
results on CPU and CUDA for uniform columns; Zipf columns use an inverse-CDF
table built once in float64 on the host and ``searchsorted``).

Workload recipes follow SURVEY.md §8(d) (table "Synthetic inputs"); the paper's
IMDB/JOB data is not available, see DESIGN.md "Inputs".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1
POINT, RANGE, SUBSET = 0, 1, 2


def _s64(c: int) -> int:
    """unsigned 64-bit constant -> signed int64 (two's complement)."""
    c &= (1 << 64) - 1
    return c - (1 << 64) if c >= (1 << 63) else c


_G = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = z + _G
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _stream_key(data_seed: int, table: str, col: str) -> int:
    h = 1469598103934665603
    for ch in f"{data_seed}/{table}/{col}".encode():
        h = ((h ^ ch) * 1099511628211) & ((1 << 64) - 1)
    return _s64(h)


def _u01(key: int, rows: torch.Tensor) -> torch.Tensor:
    """uniform double in [0, 1) from (stream key, global row index)."""
    z = _mix(_mix(rows * _C1 + key) + key)
    return _lsr(z, 11).to(torch.float64) * (1.0 / 9007199254740992.0)


_CDF_CACHE: dict = {}


def _zipf_cdf(s: float, n: int, device) -> torch.Tensor:
    """P(rank k) ∝ k^-s, k = 1..n (SURVEY.md §8(c) reading 17).  float64, host-built."""
    k = (float(s), int(n), str(device))
    if k not in _CDF_CACHE:
        host_key = (float(s), int(n), "cpu")
        if host_key not in _CDF_CACHE:
            p = np.arange(1, n + 1, dtype=np.float64) ** (-float(s))
            c = np.cumsum(p)
            c /= c[-1]
            _CDF_CACHE[host_key] = torch.from_numpy(c)
        _CDF_CACHE[k] = _CDF_CACHE[host_key].to(device)
    return _CDF_CACHE[k]


@dataclass
class Col:
    name: str
    dtype: str                 # "int32" | "int64"
    dist: tuple                # ("uniform", lo, hi) | ("zipf", s, N) | ("rowid",)
    domain: int = 0            # values lie in [0, domain) (0 = not stated); filled by Table



@dataclass
class Pred:
    col: str
    kind: int                  # POINT | RANGE | SUBSET
    lo: int = 0
    hi: int = 0
    set_values: list | None = None
    point_from_row0: bool = False   # POINT constant = value of the column at global row 0


@dataclass
class Table:
    name: str
    n_rows: int
    cols: list
    preds: list = field(default_factory=list)

    def col(self, name: str) -> Col:
        return next(c for c in self.cols if c.name == name)

    def __post_init__(self):
        # value-domain statement of each generated column (a property of the generator)
        for c in self.cols:
            if c.dist[0] == "rowid":
                c.domain = self.n_rows
            elif c.dist[0] == "uniform" and c.dist[1] >= 0:
                c.domain = int(c.dist[2])
            elif c.dist[0] == "zipf":
                c.domain = int(c.dist[2])


@dataclass
class Sketch:
    table: str
    key_cols: list             # 1 or 2 column names
    edge_ids: list             # canonical edge ids, same length as key_cols
    d: int
    w: list


@dataclass
class Workload:
    name: str
    tables: list
    edges: list                # (edge_id, table_u, table_v)
    sketches: list
    master_seed: int = 42
    data_seed: int = 210202440
    kind: str = "graph"        # "graph" (estimate + plan) | "selfjoin" (C4)

    def table(self, name: str) -> Table:
        return next(t for t in self.tables if t.name == name)

    def sketches_of(self, name: str) -> list:
        return [s for s in self.sketches if s.table == name]

    @property
    def total_rows(self) -> int:
        return sum(t.n_rows for t in self.tables)


def edge_id(a: str, b: str) -> str:
    """canonical id: the two alias.column strings sorted, joined by '|'."""
    x, y = sorted([a, b])
    return f"{x}|{y}"


def shard_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """contiguous row ranges, remainder spread one row each over the low ranks."""
    base, rem = divmod(n_rows, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def _gen_column(ws: Workload, t: Table, c: Col, r0: int, r1: int, device, chunk: int = 1 << 25) -> torch.Tensor:
    dt = torch.int32 if c.dtype == "int32" else torch.int64
    out = torch.empty(r1 - r0, dtype=dt, device=device)
    key = _stream_key(ws.data_seed, t.name, c.name)
    for s in range(r0, r1, chunk):
        e = min(r1, s + chunk)
        rows = torch.arange(s, e, dtype=torch.int64, device=device)
        if c.dist[0] == "rowid":
            v = rows
        elif c.dist[0] == "uniform":
            lo, hi = int(c.dist[1]), int(c.dist[2])
            u = _u01(key, rows)
            v = torch.clamp((u * float(hi - lo)).floor().to(torch.int64), max=hi - lo - 1) + lo
        elif c.dist[0] == "zipf":
            s_, n = float(c.dist[1]), int(c.dist[2])
            u = _u01(key, rows)
            if s_ == 0.0:
                v = torch.clamp((u * float(n)).floor().to(torch.int64), max=n - 1)
            else:
                cdf = _zipf_cdf(s_, n, device)
                v = torch.clamp(torch.searchsorted(cdf, u, right=True), max=n - 1)
        else:
            raise ValueError(c.dist)
        out[s - r0:e - r0] = v.to(dt)
        del rows, v
    return out


def subset_values(ws: Workload, t: Table, p: Pred, count: int, domain: int) -> list:
    """`count` seeded distinct values in [0, domain) for a SUBSET predicate."""
    key = _stream_key(ws.data_seed, t.name, "subset:" + p.col)
    vals, seen, i = [], set(), 0
    while len(vals) < count:
        rows = torch.arange(i, i + 4 * count, dtype=torch.int64)
        cand = (_u01(key, rows) * domain).floor().to(torch.int64).tolist()
        for v in cand:
            if v not in seen:
                seen.add(v)
                vals.append(v)
                if len(vals) == count:
                    break
        i += 4 * count
    return sorted(vals)


def generate_table(ws: Workload, name: str, device="cpu", rank: int = 0, world: int = 1) -> dict:
    """Columns of table `name` for this rank's row shard: {col: tensor}."""
    t = ws.table(name)
    r0, r1 = shard_range(t.n_rows, rank, world)
    return {c.name: _gen_column(ws, t, c, r0, r1, device) for c in t.cols}


def resolve_preds(ws: Workload, name: str, device="cpu") -> list:
    """Predicates of table `name` with data-dependent constants filled in:
    list of (col, kind, lo, hi, set_values)."""
    t = ws.table(name)
    out = []
    for p in t.preds:
        lo, hi = p.lo, p.hi
        if p.point_from_row0:
            c = next(c for c in t.cols if c.name == p.col)
            lo = hi = int(_gen_column(ws, t, c, 0, 1, "cpu")[0])
        out.append((p.col, p.kind, lo, hi, p.set_values))
    return out


# --------------------------------------------------------------------------
# BASELINE.json configs (SURVEY.md §8(d) "Synthetic inputs")
# --------------------------------------------------------------------------

def c1(scale: float = 1.0) -> Workload:
    n = max(1, int(100_000 * scale))
    e = edge_id("R.key", "S.key")
    R = Table("R", n, [Col("key", "int32", ("uniform", 0, 10000)), Col("attr", "int32", ("uniform", 1900, 2025))],
              [Pred("attr", RANGE, 2011, INT64_MAX)])                      # attr > 2010
    S = Table("S", n, [Col("key", "int32", ("uniform", 0, 10000))])
    return Workload("C1", [R, S], [(e, "R", "S")],
                    [Sketch("R", ["key"], [e], 5, [1024]), Sketch("S", ["key"], [e], 5, [1024])],
                    data_seed=210202440 + 0)


def c2(scale: float = 1.0) -> Workload:
    n = max(1, int(10_000_000 * scale))
    dom = max(16, int(1_000_000 * min(1.0, scale * 10)))
    e1, e2 = edge_id("A.key1", "B.key1"), edge_id("B.key2", "C.key2")
    z = ("zipf", 1.0, dom)
    A = Table("A", n, [Col("key1", "int32", z), Col("attr", "int32", ("uniform", 0, 100))],
              [Pred("attr", RANGE, 20, 29)])
    B = Table("B", n, [Col("key1", "int32", z), Col("key2", "int32", z)])
    C = Table("C", n, [Col("key2", "int32", z)])
    sk = [Sketch("A", ["key1"], [e1], 5, [1024]), Sketch("B", ["key1"], [e1], 5, [1024]),
          Sketch("B", ["key2"], [e2], 5, [1024]), Sketch("C", ["key2"], [e2], 5, [1024]),
          Sketch("B", ["key1", "key2"], [e1, e2], 5, [256, 256])]
    return Workload("C2", [A, B, C], [(e1, "A", "B"), (e2, "B", "C")], sk, data_seed=210202440 + 1)


def c3(scale: float = 1.0, w: int = 4096, d: int = 7) -> Workload:
    def sz(n):
        return max(8, int(n * scale))
    nT, nMK, nCI, nK, nN = sz(2_500_000), sz(4_500_000), sz(36_000_000), sz(134_000), sz(4_100_000)
    zK, zT, zN = ("zipf", 1.2, nK), ("zipf", 1.2, nT), ("zipf", 1.2, nN)
    e1 = edge_id("K.id", "MK.kid")
    e2 = edge_id("T.id", "MK.mid")
    e3 = edge_id("T.id", "CI.mid")
    e4 = edge_id("CI.mid", "MK.mid")
    e5 = edge_id("N.id", "CI.pid")
    K = Table("K", nK, [Col("id", "int32", ("rowid",)), Col("attr", "int32", ("uniform", 0, 100_000))],
              [Pred("attr", POINT, point_from_row0=True)])
    T = Table("T", nT, [Col("id", "int32", ("rowid",)), Col("attr", "int32", ("uniform", 0, 100))],
              [Pred("attr", RANGE, 0, 19)])
    MK = Table("MK", nMK, [Col("kid", "int32", zK), Col("mid", "int32", zT)])
    CI = Table("CI", nCI, [Col("mid", "int32", zT), Col("pid", "int32", zN)])
    N = Table("N", nN, [Col("id", "int32", ("rowid",)), Col("attr", "int32", ("uniform", 0, 1_000_000))])
    ws = Workload("C3", [T, MK, CI, K, N],
                  [(e1, "K", "MK"), (e2, "MK", "T"), (e3, "CI", "T"), (e4, "CI", "MK"), (e5, "CI", "N")],
                  [Sketch("K", ["id"], [e1], d, [w]),
                   Sketch("MK", ["kid"], [e1], d, [w]), Sketch("MK", ["mid"], [e2], d, [w]),
                   Sketch("MK", ["mid"], [e4], d, [w]),
                   Sketch("T", ["id"], [e2], d, [w]), Sketch("T", ["id"], [e3], d, [w]),
                   Sketch("CI", ["mid"], [e3], d, [w]), Sketch("CI", ["mid"], [e4], d, [w]),
                   Sketch("CI", ["pid"], [e5], d, [w]),
                   Sketch("N", ["id"], [e5], d, [w])],
                  data_seed=210202440 + 2)
    pN = Pred("attr", SUBSET)
    pN.set_values = subset_values(ws, N, pN, 1000, 1_000_000)
    N.preds = [pN]
    return ws


def c3t(scale: float = 1.0, w: int = 4096, d: int = 7, wt: int = 64) -> Workload:
    """C3 with partitioned sketches for its multi-join tables (PAPER.md:225
    "a table with 3 joins has a 3-D tensor as its sketch, with one dimension for every join
    attribute"): MK and CI get d x wt^3 tensors over their three edges, T a wt x wt matrix over
    its two; dimensions in canonical edge order.  Same tables, data and 1-D sketches as C3."""
    ws = c3(scale=scale, w=w, d=d)
    e = {nm: ed for ed, u, v in ws.edges for nm in [(u, v)]}
    e1, e2, e3, e4, e5 = e[("K", "MK")], e[("MK", "T")], e[("CI", "T")], e[("CI", "MK")], e[("CI", "N")]
    col_of = {("MK", e1): "kid", ("MK", e2): "mid", ("MK", e4): "mid",
              ("CI", e3): "mid", ("CI", e4): "mid", ("CI", e5): "pid", ("T", e2): "id", ("T", e3): "id"}
    for t, es in [("MK", [e1, e2, e4]), ("CI", [e3, e4, e5]), ("T", [e2, e3])]:
        es = sorted(es)
        ws.sketches.append(Sketch(t, [col_of[(t, x)] for x in es], es, d, [wt] * len(es)))
    ws.name = "C3t"
    return ws


def c4(scale: float = 1.0, w: int = 16384, d: int = 9) -> Workload:
    n = max(1, int(1_000_000_000 * scale))
    dom = 100_000_000
    z = ("zipf", 1.5, dom)
    cols = [Col("key1", "int64", z), Col("key2", "int64", z)] + \
           [Col(f"p{i}", "int32", ("uniform", 0, 1000)) for i in (1, 2, 3)]
    F = Table("F", n, cols, [Pred(f"p{i}", RANGE, INT64_MIN, 367) for i in (1, 2, 3)])   # p_i < 368
    e1, e2 = edge_id("F.key1", "D1.key"), edge_id("F.key2", "D2.key")
    return Workload("C4", [F], [], [Sketch("F", ["key1"], [e1], d, [w]), Sketch("F", ["key2"], [e2], d, [w])],
                    data_seed=210202440 + 3, kind="selfjoin")


C5_DISTS = [("zipf", 0.0), ("zipf", 0.5), ("zipf", 1.0), ("zipf", 2.0)]


def c5(scale: float = 1.0, cycle: bool = False, w: int = 1024, wm: int = 512, d: int = 5,
       n_tables: int = 10) -> Workload:
    n = max(1, int(200_000_000 * scale))
    dom = 1_000_000
    tables, edges, sk = [], [], []
    names = [f"T{i}" for i in range(1, n_tables + 1)]
    links = [(i, i + 1) for i in range(n_tables - 1)] + ([(n_tables - 1, 0)] if cycle else [])
    for i, nm in enumerate(names):
        s = C5_DISTS[i % 4][1]
        dist = ("zipf", s, dom)
        cols = []
        has_a = i > 0 or cycle
        has_b = i < n_tables - 1 or cycle
        if has_a:
            cols.append(Col("a", "int32", dist))
        if has_b:
            cols.append(Col("b", "int32", dist))
        cols.append(Col("p", "int32", ("uniform", 0, 1_000_000)))
        sel = 1e-4 * 5000 ** (i / (n_tables - 1))
        hi = int(math.ceil(sel * 1_000_000)) - 1
        tables.append(Table(nm, n, cols, [Pred("p", RANGE, 0, hi)]))
    for (i, j) in links:
        eid = edge_id(f"{names[i]}.b", f"{names[j]}.a")
        edges.append((eid, names[i], names[j]))
        sk.append(Sketch(names[i], ["b"], [eid], d, [w]))
        sk.append(Sketch(names[j], ["a"], [eid], d, [w]))
    for t in tables:
        inc = sorted([(e, (u == t.name)) for e, u, v in edges if t.name in (u, v)])
        if len(inc) == 2:
            keycols = ["b" if is_u else "a" for e, is_u in inc]
            sk.append(Sketch(t.name, keycols, [e for e, _ in inc], d, [wm, wm]))
    return Workload("C5-cycle" if cycle else "C5-chain", tables, edges, sk, data_seed=210202440 + 4)


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C3t": c3t, "C4": c4, "C5": c5}
