"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star): counters and survivor counts bit-exact (int64);
estimates exact per row (both sides compute E_r exactly; the median is rounded
once to fp64, so fp64 values are compared with ==, which is stricter than the
north-star tolerance rel 1e-12); greedy join order identical.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2102_02440_b200 as pb
from paper_2102_02440_b200.query import QueryRun

pytestmark = pytest.mark.gpu

I64MIN, I64MAX = -(1 << 63), (1 << 63) - 1


def _dev():
    return torch.device("cuda", 0)


def _rand_cols(n, seed):
    rng = np.random.default_rng(seed)
    k32 = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    k64 = rng.integers(I64MIN, I64MAX, n, dtype=np.int64, endpoint=True)
    if n > 10:
        k32[:4] = [-2**31, 2**31 - 1, 0, -1]
        k64[:6] = [I64MIN, I64MAX, 0, -1, (1 << 61) - 1, 1 << 61]
    zk = rng.zipf(1.3, n).astype(np.int64) % 5000          # skewed key
    p = rng.integers(0, 100, n).astype(np.int32)
    s = rng.integers(0, 50, n).astype(np.int64)
    return {"k32": k32, "k64": k64, "zk": zk, "p": p, "s": s}


def _to_dev(cols):
    return {k: torch.from_numpy(v).to(_dev()) for k, v in cols.items()}


TARGETS = [  # (key cols, d, w, edge ids)
    (["k32"], 5, [1024], ["A.k32|B.x"]),
    (["k64"], 3, [64], ["A.k64|C.y"]),
    (["zk"], 7, [4096], ["A.zk|D.z"]),
    (["k32", "k64"], 3, [32, 16], ["A.k32|B.x", "A.k64|C.y"]),
    (["zk", "k32"], 5, [64, 128], ["A.k32|B.x", "A.zk|D.z"]),
]


def _gpu_build(cols, preds, targets, master=42, calls=1, domains=None):
    names = list(cols)
    dom = [domains.get(c, 0) for c in names] if domains else None
    dcols = _to_dev(cols)
    sks = [pb.Sketch(d, w, e, master, _dev()) for (_, d, w, e) in targets]
    surv = torch.zeros(1, dtype=torch.int64, device=_dev())
    n = len(cols[names[0]])
    cuts = np.linspace(0, n, calls + 1).astype(int)
    for a, b in zip(cuts[:-1], cuts[1:]):
        sub = [dcols[c][a:b].contiguous() for c in names]
        pr = [(names.index(p[0]),) + tuple(p[1:]) for p in preds]
        tg = [(sk, [names.index(k) for k in t[0]]) for sk, t in zip(sks, targets)]
        pb.sketch_update_filtered(sub, int(b - a), pr, tg, survivors=surv, domains=dom)
    torch.cuda.synchronize()
    return [sk.counters.cpu().numpy() for sk in sks], int(surv.item())


def _oracle_build(cols, preds, targets, master=42):
    mask, cnt = oracle.filter_mask(cols, preds)
    outs = []
    for keys, d, w, e in targets:
        outs.append(oracle.build([cols[k] for k in keys], mask, d, w, e, master=master))
    return outs, cnt


PRED_SETS = [
    [],
    [("p", pb.RANGE, 10, 69)],
    [("p", pb.RANGE, 10, 69), ("s", pb.SUBSET, 0, 0, [1, 3, 5, 7, 11, 13, 49, 1000])],
    [("s", pb.POINT, 7, 7)],
    [("k64", pb.RANGE, I64MIN, 0), ("p", pb.RANGE, 0, I64MAX)],
    [("s", pb.SUBSET, 0, 0, [])],                       # nothing qualifies
    [("p", pb.POINT, 1000, 1000)],                      # nothing qualifies
]


@pytest.fixture(params=["optimised", "generic"])
def scan_mode(request, monkeypatch):
    """Run build tests through both kernels: the persistent TMA scan and the generic one."""
    if request.param == "generic":
        monkeypatch.setenv("COMPASS_SCAN", "generic")
    else:
        monkeypatch.delenv("COMPASS_SCAN", raising=False)
    return request.param


@pytest.mark.parametrize("n", [0, 1, 31, 4097, 100_003, 1_000_000])
@pytest.mark.parametrize("pi", range(len(PRED_SETS)))
def test_build_parity(n, pi, scan_mode):
    cols = _rand_cols(n, 1000 + n + pi)
    preds = PRED_SETS[pi]
    g, gs = _gpu_build(cols, preds, TARGETS)
    o, os_ = _oracle_build(cols, preds, TARGETS)
    assert gs == os_
    for a, b in zip(g, o):
        assert np.array_equal(a, b)


# key-domain hints: zk is in [0, 5000) (histogram mode), k32's hint 1000 is violated by most
# rows (out-of-domain fallback), p/s hints on predicate-only columns are ignored
DOMAINS = [None, {"zk": 5000, "k32": 1000, "p": 100, "s": 50}, {"zk": 4096}]


@pytest.mark.parametrize("n", [1, 4097, 1_000_000])
@pytest.mark.parametrize("di", range(1, len(DOMAINS)))
@pytest.mark.parametrize("pi", [0, 1, 2, 5])
def test_build_parity_domain_hints(n, di, pi):
    cols = _rand_cols(n, 2000 + n + pi)
    preds = PRED_SETS[pi]
    g, gs = _gpu_build(cols, preds, TARGETS, domains=DOMAINS[di])
    o, os_ = _oracle_build(cols, preds, TARGETS)
    assert gs == os_
    for a, b in zip(g, o):
        assert np.array_equal(a, b)


# single-width key targets under int32 range predicates select the specialised scan
# (KW = 4 or 8: survivors gathered straight from the ballots); the same inputs through the
# generic variant (COMPASS_SCAN_KW0) and the grid-stride kernel must give the same counters.
# Selectivities 1% .. 100% cover the ring-full rounds (a 128-row slice with > 64 survivors).
KW_TARGETS = {
    4: [(["k32"], 5, [1024], ["A.k32|B.x"]), (["p2"], 3, [64], ["A.p2|C.y"]),
        (["k32", "p2"], 3, [32, 16], ["A.k32|B.x", "A.p2|C.y"])],
    8: [(["k64"], 3, [64], ["A.k64|C.y"]), (["zk"], 9, [16384], ["A.zk|D.z"]),
        (["zk", "k64"], 5, [64, 128], ["A.k64|C.y", "A.zk|D.z"])],
}


@pytest.mark.parametrize("kw", [4, 8])
@pytest.mark.parametrize("hi", [0, 36, 49, 99])
@pytest.mark.parametrize("variant", ["kw", "kw0", "generic"])
@pytest.mark.parametrize("n", [31, 100_003, 1_000_000])
def test_build_parity_specialised_scan(kw, hi, variant, n, monkeypatch):
    if variant == "kw0":
        monkeypatch.setenv("COMPASS_SCAN_KW0", "1")
    elif variant == "generic":
        monkeypatch.setenv("COMPASS_SCAN", "generic")
    cols = _rand_cols(n, 3000 + n + hi)
    cols["p2"] = np.random.default_rng(n).integers(-50, 50, n).astype(np.int32)
    preds = [("p", pb.RANGE, 0, hi), ("p2", pb.RANGE, -50, 49)]
    g, gs = _gpu_build(cols, preds, KW_TARGETS[kw])
    o, os_ = _oracle_build(cols, preds, KW_TARGETS[kw])
    assert gs == os_
    for a, b in zip(g, o):
        assert np.array_equal(a, b)


def test_build_parity_global_atomic_path_and_skew(scan_mode):
    """A sketch too large for shared memory (C4 shape d=9, w=16384) next to a privatised one."""
    cols = _rand_cols(3_000_001, 77)
    tg = [(["zk"], 9, [16384], ["F.key1|D1.key"]), (["k64"], 9, [16384], ["F.key2|D2.key"]), (["k32"], 5, [1024], ["x|y"])]
    preds = [("p", pb.RANGE, I64MIN, 36)]
    g, gs = _gpu_build(cols, preds, tg)
    o, os_ = _oracle_build(cols, preds, tg)
    assert gs == os_ and all(np.array_equal(a, b) for a, b in zip(g, o))


def test_sharded_calls_accumulate_and_merge_is_exact(scan_mode):
    cols = _rand_cols(200_000, 5)
    preds = PRED_SETS[2]
    one, s1 = _gpu_build(cols, preds, TARGETS, calls=1)
    many, s8 = _gpu_build(cols, preds, TARGETS, calls=8)
    assert s1 == s8 and all(np.array_equal(a, b) for a, b in zip(one, many))
    # sketch_merge of two independently built halves
    names = list(cols)
    dcols = _to_dev(cols)
    half = 100_000
    sks = []
    for a, b in ((0, half), (half, 200_000)):
        sk = pb.Sketch(5, [1024], ["A.k32|B.x"], 42, _dev())
        pb.sketch_update_filtered([dcols[c][a:b].contiguous() for c in names], b - a,
                                  [(names.index("p"), pb.RANGE, 10, 69)], [(sk, [names.index("k32")])])
        sks.append(sk)
    pb.sketch_merge(sks[0], sks[1])
    full = oracle.build([cols["k32"]], oracle.filter_mask(cols, [("p", pb.RANGE, 10, 69)])[0], 5, [1024], ["A.k32|B.x"])
    assert np.array_equal(sks[0].counters.cpu().numpy(), full)
    other = pb.Sketch(5, [1024], ["A.k32|B.y"], 42, _dev())
    with pytest.raises(pb.SkError) as ei:
        pb.sketch_merge(sks[0], other)
    assert ei.value.status == pb.SK_EMISMATCH


def test_invalid_arguments_fail_loudly():
    with pytest.raises(pb.SkError) as ei:
        pb.Sketch(4, [1024], ["a|b"], 42, _dev())
    assert ei.value.status == pb.SK_EINVAL
    with pytest.raises(pb.SkError):
        pb.Sketch(5, [1000], ["a|b"], 42, _dev())
    with pytest.raises(pb.SkError):
        pb.Sketch(5, [64, 64], ["z|z", "a|a"], 42, _dev())   # dims not in canonical order


# ------------------------------------------------------------------ estimates on random networks
def _random_graph(rng, topo, w, d, vmax, mat_prob=0.5):
    T = 1 + max(max(e) for e in topo)
    names = [f"t{i}" for i in range(T)]
    eids = [f"{names[u]}.c{i}|{names[v]}.c{i}" for i, (u, v) in enumerate(topo)]
    widths = {e: int(w * 2 ** rng.integers(0, 2)) for e in eids}
    vec_np, mat_np = {}, {}
    for i, (u, v) in enumerate(topo):
        for t in (u, v):
            vec_np[(names[t], eids[i])] = rng.integers(-vmax, vmax + 1, (d, widths[eids[i]])).astype(np.int64)
    for t in range(T):
        inc = sorted(eids[i] for i, e in enumerate(topo) if t in e)
        if len(inc) == 2 and rng.random() < mat_prob:
            mat_np[(names[t], tuple(inc))] = rng.integers(-vmax, vmax + 1, (d, w, w)).astype(np.int64)
    og = oracle.Graph({n: int(rng.integers(1, 1000)) for n in names}, [(eids[i], names[u], names[v]) for i, (u, v) in enumerate(topo)],
                      vec_np, mat_np)
    sk = {}
    for key, arr in vec_np.items():
        s = pb.Sketch(d, [arr.shape[1]], [key[1]], 42, _dev())
        s.counters.copy_(torch.from_numpy(arr))
        sk[key] = s
    mats = []
    for (t, inc), arr in mat_np.items():
        s = pb.Sketch(d, [w, w], list(inc), 42, _dev())
        s.counters.copy_(torch.from_numpy(arr))
        mats.append((names.index(t), eids.index(inc[0]), eids.index(inc[1]), s))
    edges = [(u, v, sk[(names[u], eids[i])], sk[(names[v], eids[i])]) for i, (u, v) in enumerate(topo)]
    jg = pb.JoinGraph(names, [og.tables[n] for n in names], edges, mats)
    return og, jg, (sk, mats)


TOPOS = [
    [(0, 1)], [(0, 1), (1, 2)], [(0, 1), (1, 2), (2, 3), (3, 4)], [(0, 1), (1, 2), (0, 2)],
    [(1, 0), (0, 2), (1, 2), (2, 3), (1, 4)], [(0, 1), (0, 2), (0, 3)], [(0, 1), (1, 2), (2, 3), (3, 0)],
    [(2, 1), (0, 1), (3, 1), (2, 0)], [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)],
]


ENUM_CASES = [("greedy", 1, True), ("full-greedy", 1, True), ("limit", 10, True), ("limit", 2, True),
              ("exhaustive", 0, True), ("exhaustive", 0, False)]


def _check_enumerate(og, jg, est_cache=None):
    """plan_enumerate (Algorithm 1) through the C-ABI == the oracle's, every mode: same
    order, per-prefix cards, cost and traversal counters (both sides see identical estimates)."""
    cache = dict(est_cache or {})

    def est(S):
        if S not in cache:
            cache[S] = oracle.estimate(og, S)[0]
        return cache[S]
    for mode, mp, prune in ENUM_CASES:
        o_order, o_pre, o_cost, o_st = oracle.plan_enumerate(og, mode=mode, max_plans=mp, prune=prune, est_fn=est)
        order, pre, cost, st = jg.plan_enumerate(mode=mode, max_plans=mp, prune=prune)
        assert (order, pre, cost) == (o_order, o_pre, o_cost), (mode, mp, prune)
        assert st["plans_completed"] == o_st["plans_completed"], (mode, mp, prune)
        if mode != "greedy":
            assert st["prunes"] == o_st["prunes"], (mode, mp, prune)


@pytest.fixture(params=["default", "crt"])
def est_engine(request, monkeypatch):
    """Estimates through the default engine (exact int128 contraction where the bound fits,
    int128 dot products for two-way sub-plans) and through the CRT engine alone."""
    if request.param == "crt":
        monkeypatch.setenv("COMPASS_EST_CRT_ONLY", "1")
    else:
        monkeypatch.delenv("COMPASS_EST_CRT_ONLY", raising=False)
    return request.param


@pytest.mark.parametrize("ti", range(len(TOPOS)))
def test_estimates_equal_oracle_on_random_networks(ti, est_engine):
    rng = np.random.default_rng(300 + ti)
    for trial in range(3):
        og, jg, keep = _random_graph(rng, TOPOS[ti], w=8, d=3, vmax=[3, 1000, 2**40][trial])
        for s in oracle.connected_subplans(og):
            want = oracle.estimate_rows(og, s)
            got = jg.estimate_join_exact(s)
            assert got == want, (ti, trial, s)
            est, rows = jg.estimate_join(s)
            assert est == float(oracle.median_odd(want)) and rows == [float(v) for v in want]
        assert tuple(jg.plan_greedy()) == tuple(oracle.plan_greedy(og))
        _check_enumerate(og, jg)


# ------------------------------------------------------------------ workloads C1-C5
def _run_workload(ws, device=None):
    device = device or _dev()
    run = QueryRun(ws, device)
    data_d, data_h, preds = {}, {}, {}
    for t in ws.tables:
        data_d[t.name] = datagen.generate_table(ws, t.name, device)
        data_h[t.name] = {k: v.cpu().numpy() for k, v in data_d[t.name].items()}
        preds[t.name] = datagen.resolve_preds(ws, t.name)
    run.build(data_d, preds)
    torch.cuda.synchronize()
    return run, data_h, preds


def _oracle_workload(ws, data_h, preds):
    vec, mat, surv = {}, {}, {}
    for t in ws.tables:
        mask, cnt = oracle.filter_mask(data_h[t.name], preds[t.name])
        surv[t.name] = cnt
        for s in ws.sketches_of(t.name):
            arr = oracle.build([data_h[t.name][k] for k in s.key_cols], mask, s.d, s.w, s.edge_ids, master=ws.master_seed)
            if len(s.w) == 1:
                vec[(t.name, s.edge_ids[0])] = arr
            else:
                mat[(t.name, tuple(s.edge_ids))] = arr
    return oracle.Graph(surv, ws.edges, vec, mat), surv


def _check_counters(ws, run, og, surv):
    assert run.survivors.tolist() == [surv[t.name] for t in ws.tables]
    for s, sk in zip(ws.sketches, run.sketches):
        want = og.vec[(s.table, s.edge_ids[0])] if len(s.w) == 1 else og.mat[(s.table, tuple(s.edge_ids))]
        assert np.array_equal(sk.counters.cpu().numpy(), want), (s.table, s.edge_ids)


def test_c1_end_to_end(est_engine):
    ws = datagen.c1()
    run, data_h, preds = _run_workload(ws)
    og, surv = _oracle_workload(ws, data_h, preds)
    _check_counters(ws, run, og, surv)
    jg = run.graph()
    assert jg.estimate_join_exact(("R", "S")) == oracle.estimate_rows(og, ("R", "S"))
    est, _ = jg.estimate_join(("R", "S"))
    assert est == oracle.estimate(og, ("R", "S"))[0]
    assert list(jg.plan_greedy()[0]) == oracle.plan_greedy(og)[0]
    _check_enumerate(og, jg)


def _all_subplans_match(ws, run, og, rows=None):
    jg = run.graph()
    for s in oracle.connected_subplans(og):
        want = oracle.estimate_rows(og, s, rows=rows)
        got = jg.estimate_join_exact(s)
        if rows is not None:
            got = [got[r] for r in rows]
        assert got == want, s
    return jg


def test_c2_scaled_chain_parity():
    ws = datagen.c2(scale=0.01)
    run, data_h, preds = _run_workload(ws)
    og, surv = _oracle_workload(ws, data_h, preds)
    _check_counters(ws, run, og, surv)
    jg = _all_subplans_match(ws, run, og)
    order, pre, cost = jg.plan_greedy()
    o_order, o_pre, o_cost = oracle.plan_greedy(og)
    assert order == o_order and pre == o_pre and cost == o_cost
    _check_enumerate(og, jg)


def test_c3_scaled_parity_all_14_subplans_and_plan(est_engine):
    ws = datagen.c3(scale=0.005, w=256)
    run, data_h, preds = _run_workload(ws)
    og, surv = _oracle_workload(ws, data_h, preds)
    _check_counters(ws, run, og, surv)
    jg = _all_subplans_match(ws, run, og)
    assert tuple(jg.plan_greedy()) == tuple(oracle.plan_greedy(og))
    _check_enumerate(og, jg)


@pytest.mark.parametrize("cycle", [False, True])
def test_c5_scaled_parity_all_subplans_and_plan(cycle):
    ws = datagen.c5(scale=2e-4, cycle=cycle, w=128, wm=64)
    run, data_h, preds = _run_workload(ws)
    og, surv = _oracle_workload(ws, data_h, preds)
    _check_counters(ws, run, og, surv)
    jg = _all_subplans_match(ws, run, og)
    assert tuple(jg.plan_greedy()) == tuple(oracle.plan_greedy(og))
    _check_enumerate(og, jg)


def test_c3_full_width_triangle_sampled_row(est_engine):
    """C3 at its full sketch shape (d=7, w=4096), rows scaled: the triangle and the
    5-table sub-plan, row 0 only (the oracle's cost is O(w^2 log w) big-int ops)."""
    ws = datagen.c3(scale=0.01)
    run, data_h, preds = _run_workload(ws)
    og, surv = _oracle_workload(ws, data_h, preds)
    _check_counters(ws, run, og, surv)
    jg = run.graph()
    for s in [("CI", "MK", "T"), ("CI", "K", "MK", "N", "T")]:
        assert jg.estimate_join_exact(s)[0] == oracle.estimate_rows(og, s, rows=[0])[0]


# ------------------------------------------------------------------ exact join sizes (accuracy, §8(f) 2)
XSHAPES = [[("A", "B", "k", "k")], [("A", "B", "k", "k"), ("B", "C", "j", "j"), ("C", "D", "k", "j")],
           [("A", "B", "k", "k"), ("A", "C", "j", "k"), ("A", "D", "k", "j"), ("D", "E", "k", "k")]]


def _xtables(rng, names, n, dom):
    T = {}
    for t in names:
        cols = {"k": rng.integers(0, dom, n).astype(np.int32), "j": rng.integers(0, dom, n).astype(np.int64),
                "p": rng.integers(0, 100, n).astype(np.int32)}
        preds = [[], [("p", pb.RANGE, 5, 90)], [("p", pb.SUBSET, 0, 0, list(range(0, 100, 3)))],
                 [("p", pb.POINT, 7, 7)]][int(rng.integers(0, 4))]
        T[t] = (cols, preds)
    return T


def _x_gpu_args(T, E, names, dom):
    tables, cpos = [], {}
    for t in names:
        cols, preds = T[t]
        cn = list(cols)
        cpos[t] = {c: i for i, c in enumerate(cn)}
        tables.append(([torch.from_numpy(cols[c]).to(_dev()) for c in cn],
                       [(cn.index(p[0]),) + tuple(p[1:]) for p in preds]))
    edges = [(names.index(u), names.index(v), cpos[u][cu], cpos[v][cv], 0, dom) for u, v, cu, cv in E]
    return tables, edges


@pytest.mark.parametrize("si", range(len(XSHAPES)))
def test_exact_join_size_equals_oracle(si):
    """Every acyclic connected sub-plan of random trees (counts far beyond 2^64 on the larger
    cases: several CRT moduli) — exact decimal equality with the oracle's Python integers."""
    import evaluation as accuracy
    rng = np.random.default_rng(400 + si)
    E = XSHAPES[si]
    names = sorted({x for e in E for x in e[:2]})
    for n, dom in [(1, 4), (2000, 16), (50_000, 64)]:
        T = _xtables(rng, names, n, dom)
        tables, edges = _x_gpu_args(T, E, names, dom)
        for sub in accuracy.acyclic_connected_subplans(names, edges, min_size=1):
            got = pb.exact_join_size(tables, edges, sum(1 << names.index(t) for t in sub))
            assert got == oracle.exact_join_size(T, E, sub), (si, n, sub)


XCYCLES = [
    [("A", "B", "k", "k"), ("A", "C", "k", "k"), ("B", "C", "k", "k")],                       # one-key triangle
    [("A", "B", "k", "j"), ("B", "C", "k", "j"), ("C", "A", "k", "j")],                       # genuine triangle
    [("A", "B", "j", "k"), ("B", "C", "j", "k"), ("C", "D", "j", "k"), ("D", "A", "j", "k")],  # 4-cycle
    [("A", "B", "k", "k"), ("A", "B", "j", "j"), ("B", "C", "k", "j")],                       # parallel edges
    [("K", "M", "k", "j"), ("M", "T", "k", "k"), ("C", "T", "k", "k"), ("C", "M", "k", "k"), ("C", "N", "j", "k")],
]


@pytest.mark.parametrize("si", range(len(XCYCLES)))
def test_exact_join_size_cyclic_equals_oracle(si):
    """Every connected sub-plan of graphs with cycles (implied edges dropped, genuine cycles
    conditioned on one edge) — exact equality with the oracle's hash join with multiplicities
    (oracle.exact_join_size_any, pinned by the nested-loop definition)."""
    import evaluation as accuracy
    rng = np.random.default_rng(700 + si)
    E = XCYCLES[si]
    names = sorted({x for e in E for x in e[:2]})
    for n, dom in [(1, 4), (300, 8), (5000, 32)]:
        T = _xtables(rng, names, n, dom)
        tables, edges = _x_gpu_args(T, E, names, dom)
        for sub in accuracy.connected_subplans(names, edges, min_size=1):
            got = pb.exact_join_size(tables, edges, sum(1 << names.index(t) for t in sub))
            assert got == oracle.exact_join_size_any(T, E, sub), (si, n, sub)


def test_exact_join_size_errors():
    rng = np.random.default_rng(5)
    E = [("A", "B", "k", "k"), ("B", "C", "j", "j"), ("A", "C", "j", "k")]   # a genuine triangle
    names = ["A", "B", "C"]
    T = _xtables(rng, names, 100, 8)
    tables, edges = _x_gpu_args(T, E, names, 1 << 20)   # conditioning 2^20 keys exceeds the limit
    with pytest.raises(pb.SkError) as ei:
        pb.exact_join_size(tables, edges, 0b111)
    assert ei.value.status == pb.SK_EOVERFLOW
    tables, edges = _x_gpu_args(T, E, names, 4)          # keys in [0, 8) outside the domain [0, 4)
    with pytest.raises(pb.SkError) as ei:
        pb.exact_join_size(tables, edges, 0b011)
    assert ei.value.status == pb.SK_EINVAL


def test_c3_triangle_subplans_exact_equals_oracle():
    """The accuracy truth of C3's four triangle-bearing sub-plans (PAPER.md:39's triangle
    T-MK-CI on one key per table: the third edge is implied) at 0.5% scale."""
    import evaluation as accuracy
    ws = datagen.c3(scale=0.005, w=256)
    run, data_h, preds = _run_workload(ws)
    data_d = {t.name: {k: torch.from_numpy(v).to(_dev()) for k, v in data_h[t.name].items()} for t in ws.tables}
    tables, edges, names = accuracy.join_data(ws, data_d, preds)
    subs = [s for s in accuracy.connected_subplans(names, edges) if {"CI", "MK", "T"} <= set(s)]
    assert len(subs) == 4
    truths = accuracy.exact_counts(tables, edges, names, subs)
    T = {t.name: (data_h[t.name], preds[t.name]) for t in ws.tables}
    keycol = {(s.table, s.edge_ids[0]): s.key_cols[0] for s in ws.sketches if len(s.edge_ids) == 1}
    OE = [(u, v, keycol[(u, e)], keycol[(v, e)]) for e, u, v in ws.edges]
    for s in subs:
        assert truths[s] == oracle.exact_join_size_any(T, OE, s), s


@pytest.mark.parametrize("which", ["C2", "C5", "C5-cycle", "C3"])
def test_accuracy_report_equals_oracle(which):
    """The accuracy evaluation of PAPER.md:261/294 on scaled C2 and C5-chain: GPU estimates and
    GPU exact counts give the same ratios and normalised L1 distances as the oracle's."""
    import evaluation as accuracy
    ws = {"C2": lambda: datagen.c2(scale=0.01), "C5": lambda: datagen.c5(scale=2e-4, w=128, wm=64),
          "C5-cycle": lambda: datagen.c5(scale=2e-4, w=128, wm=64, cycle=True),
          "C3": lambda: datagen.c3(scale=0.005, w=256)}[which]()
    run, data_h, preds = _run_workload(ws)
    og, surv = _oracle_workload(ws, data_h, preds)
    data_d = {t.name: {k: torch.from_numpy(v).to(_dev()) for k, v in data_h[t.name].items()} for t in ws.tables}
    tables, edges, names = accuracy.join_data(ws, data_d, preds)
    subs = accuracy.connected_subplans(names, edges)
    truths = accuracy.exact_counts(tables, edges, names, subs)
    jg = run.graph()
    ests = dict(zip(subs, jg.estimate_subplans(subs)))
    got = accuracy.report(ests, truths)
    # oracle side
    T = {t.name: (data_h[t.name], preds[t.name]) for t in ws.tables}
    keycol = {(s.table, s.edge_ids[0]): s.key_cols[0] for s in ws.sketches if len(s.edge_ids) == 1}
    OE = [(u, v, keycol[(u, e)], keycol[(v, e)]) for e, u, v in ws.edges]
    # the library declines only a genuine cycle over a key domain too large to condition (the
    # C5 10-cycle over 10^6 keys); every other sub-plan has a truth
    assert all(v is not None or (which == "C5-cycle" and len(s) == 10) for s, v in truths.items())
    o_truths = {s: (oracle.exact_join_size_any(T, OE, s) if truths[s] is not None else None) for s in subs}
    assert o_truths == truths
    known = {s: v for s, v in o_truths.items() if v is not None}
    want = oracle.accuracy_report({s: oracle.estimate(og, s)[0] for s in known}, known)
    assert got == want


@pytest.mark.parametrize("kw", [4, 8])
def test_zero_copy_key_columns_equal_device_build(kw):
    """Key columns of a filtered table read in place from pinned host memory (the e2e path):
    counters identical to the build from device columns and to the oracle."""
    n = 1_000_003
    cols = _rand_cols(n, 9000 + kw)
    cols["p2"] = np.random.default_rng(kw).integers(-50, 50, n).astype(np.int32)
    preds = [("p", pb.RANGE, 0, 36), ("p2", pb.RANGE, -50, 49)]
    targets = KW_TARGETS[kw]
    names = list(cols)
    dcols = _to_dev(cols)
    pcols = {p[0] for p in preds}
    mixed = [dcols[c] if c in pcols else torch.from_numpy(cols[c]).pin_memory() for c in names]
    sks = [pb.Sketch(d, w, e, 42, _dev()) for (_, d, w, e) in targets]
    surv = torch.zeros(1, dtype=torch.int64, device=_dev())
    pr = [(names.index(p[0]),) + tuple(p[1:]) for p in preds]
    tg = [(sk, [names.index(k) for k in t[0]]) for sk, t in zip(sks, targets)]
    pb.sketch_update_filtered(mixed, n, pr, tg, survivors=surv)
    torch.cuda.synchronize()
    g, gs = _gpu_build(cols, preds, targets)
    o, os_ = _oracle_build(cols, preds, targets)
    assert int(surv.item()) == gs == os_
    for sk, a, b in zip(sks, g, o):
        assert np.array_equal(sk.counters.cpu().numpy(), a) and np.array_equal(a, b)


def test_mapped_host_predicate_column_takes_the_generic_kernel():
    """A predicate column in pinned host memory cannot be staged by TMA: the call falls back
    to the grid-stride kernel and the counters are still exact."""
    n = 200_003
    cols = _rand_cols(n, 77)
    preds = [("p", pb.RANGE, 10, 69)]
    targets = TARGETS[:3]
    names = list(cols)
    host_or_dev = [torch.from_numpy(cols[c]).pin_memory() for c in names]
    sks = [pb.Sketch(d, w, e, 42, _dev()) for (_, d, w, e) in targets]
    surv = torch.zeros(1, dtype=torch.int64, device=_dev())
    pr = [(names.index(p[0]),) + tuple(p[1:]) for p in preds]
    tg = [(sk, [names.index(k) for k in t[0]]) for sk, t in zip(sks, targets)]
    pb.sketch_update_filtered(host_or_dev, n, pr, tg, survivors=surv)
    torch.cuda.synchronize()
    o, os_ = _oracle_build(cols, preds, targets)
    assert int(surv.item()) == os_
    for sk, b in zip(sks, o):
        assert np.array_equal(sk.counters.cpu().numpy(), b)
