"""GPU parity, round-2 additions (VERDICT r01 "Next round" item 1 and ADVICE r01):

* histogram mode with more 1-D sketches on one hinted key column than one epilogue launch
  serves (9..16 targets), including keys outside the hinted domain;
* the exact C4 kernel instance the bench times (2 int64 keys, 3 int32 ranges ->
  k_scan<2,3,8>) on a 3M-row slice of the C4 workload, against the oracle;
* the two-way estimate on caller-owned counters whose products leave int128 (the int128
  kernel must flag them and the CRT engine must give the exact value);
* estimate_join_exact on a singleton.

Bar: counters bit-exact (int64), estimates exact per row.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2102_02440_b200 as pb
from paper_2102_02440_b200.query import QueryRun

pytestmark = pytest.mark.gpu


def _dev():
    return torch.device("cuda", 0)


def _build(cols, preds, targets, domains=None):
    names = list(cols)
    dom = [domains.get(c, 0) for c in names] if domains else None
    dcols = [torch.from_numpy(cols[c]).to(_dev()) for c in names]
    sks = [pb.Sketch(d, w, e, 42, _dev()) for (_, d, w, e) in targets]
    surv = torch.zeros(1, dtype=torch.int64, device=_dev())
    pr = [(names.index(p[0]),) + tuple(p[1:]) for p in preds]
    tg = [(sk, [names.index(k) for k in t[0]]) for sk, t in zip(sks, targets)]
    pb.sketch_update_filtered(dcols, len(cols[names[0]]), pr, tg, survivors=surv, domains=dom)
    torch.cuda.synchronize()
    return [sk.counters.cpu().numpy() for sk in sks], int(surv.item())


def _oracle(cols, preds, targets):
    mask, cnt = oracle.filter_mask(cols, preds)
    return [oracle.build([cols[k] for k in keys], mask, d, w, e) for keys, d, w, e in targets], cnt


@pytest.mark.parametrize("n_targets", [8, 9, 16])
@pytest.mark.parametrize("with_pred", [False, True])
@pytest.mark.parametrize("n", [4097, 1_000_000])
@pytest.mark.parametrize("mode", ["optimised", "generic"])
def test_histogram_mode_serves_every_target(n_targets, with_pred, n, mode, monkeypatch):
    """9..16 1-D sketches on one hinted key column (scan.cu histogram epilogue runs in chunks
    of 8 targets); keys outside the hinted domain take the direct path."""
    if mode == "generic":
        monkeypatch.setenv("COMPASS_SCAN", "generic")
    rng = np.random.default_rng(n + n_targets)
    zk = (rng.zipf(1.2, n) % 5000).astype(np.int64)
    zk[::97] = 5000 + rng.integers(0, 10**6, zk[::97].shape[0])     # above the hint
    zk[::101] = -rng.integers(1, 10**9, zk[::101].shape[0])         # negative: canonical key >= 2^61 - 10^9
    cols = {"zk": zk, "p": rng.integers(0, 100, n).astype(np.int32)}
    targets = [(["zk"], (3, 5, 7)[t % 3], [(64, 256, 1024, 4096)[t % 4]], [f"A.zk|T{t}.k"]) for t in range(n_targets)]
    preds = [("p", pb.RANGE, 5, 60)] if with_pred else []
    g, gs = _build(cols, preds, targets, domains={"zk": 5000})
    o, os_ = _oracle(cols, preds, targets)
    assert gs == os_
    for t, (a, b) in enumerate(zip(g, o)):
        assert np.array_equal(a, b), f"target {t} differs"


def test_c4_bench_instance_equals_oracle(capfd, monkeypatch):
    """The kernel instance the C4 bench times: two int64 Zipf-1.5 keys, three int32 ranges
    (k_scan<NK=2, NP=3, KW=8>), d=9, w=16384, on the first 3M rows of the C4 workload
    (datagen.c4(scale=0.003): same generator, distributions and predicates)."""
    monkeypatch.setenv("COMPASS_SCAN_DEBUG", "1")
    ws = datagen.c4(scale=0.003)
    dev = _dev()
    run = QueryRun(ws, dev)
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    run.build(data, preds)
    torch.cuda.synchronize()
    err = capfd.readouterr().err
    assert "keys 2 preds 3 kw 8" in err, err
    t = ws.tables[0]
    cols = {k: v.cpu().numpy() for k, v in data[t.name].items()}
    mask, cnt = oracle.filter_mask(cols, preds[t.name])
    assert int(run.survivors[0].item()) == cnt
    for s, sk in zip(ws.sketches, run.sketches):
        ref = oracle.build([cols[k] for k in s.key_cols], mask, s.d, s.w, s.edge_ids, master=ws.master_seed)
        assert np.array_equal(sk.counters.cpu().numpy(), ref)
    # the C4 step's estimates: the self-join F2 of each key sketch, exact per row
    g = run.graph()
    for i, s in enumerate(ws.sketches):
        ref = oracle.build([cols[s.key_cols[0]]], mask, s.d, s.w, s.edge_ids, master=ws.master_seed)
        rows = g.estimate_join_exact((g.tables[2 * i], g.tables[2 * i + 1]))
        assert rows == [oracle.two_way_row(ref[r], ref[r]) for r in range(s.d)]


@pytest.mark.parametrize("mag", [1 << 40, (1 << 62) + 12345, (1 << 63) - 1])
def test_two_way_beyond_int128_is_flagged_and_exact(mag):
    """Caller-owned counters whose row dot products exceed int128: k_dot128 flags the rows and
    the CRT engine evaluates them; every row equals the exact Python-integer dot product."""
    rng = np.random.default_rng(mag % 1000)
    d, w = 3, 64
    A = rng.integers(-mag, mag, (d, w), dtype=np.int64, endpoint=True)
    B = rng.integers(-mag, mag, (d, w), dtype=np.int64, endpoint=True)
    A[0, :] = mag
    B[0, :] = -mag if mag > 0 else 0
    ca = torch.from_numpy(A).to(_dev())
    cb = torch.from_numpy(B).to(_dev())
    e = "X.k|Y.k"
    sa = pb.Sketch(d, [w], [e], 42, _dev(), counters=ca)
    sb = pb.Sketch(d, [w], [e], 42, _dev(), counters=cb)
    g = pb.JoinGraph(["X", "Y"], [1, 1], [(0, 1, sa, sb)], [])
    rows = g.estimate_join_exact(("X", "Y"))
    exact = [sum(int(a) * int(b) for a, b in zip(A[r], B[r])) for r in range(d)]
    assert rows == exact
    est, _ = g.estimate_join(("X", "Y"))
    assert est == float(sorted(exact)[(d - 1) // 2])


def test_estimate_join_exact_singleton():
    d, w = 5, 32
    e = "X.k|Y.k"
    sa = pb.Sketch(d, [w], [e], 42, _dev())
    sb = pb.Sketch(d, [w], [e], 42, _dev())
    g = pb.JoinGraph(["X", "Y"], [7, 11], [(0, 1, sa, sb)], [])
    assert g.estimate_join_exact(("Y",)) == [11] * d


@pytest.mark.slow
def test_c3_full_size_all_14_subplans_row0():
    """C3 at BASELINE.json's full size and sketch shape (47M rows, d=7, w=4096), the
    configuration bench.py --workload C3 times: counters bit-exact, and row 0 of all 14
    connected sub-plans (two-way, merged 3-/4-/5-table views, the triangle) equal to the
    oracle's exact value (the oracle is pinned at this width by tests/test_oracle_fullwidth.py)."""
    ws = datagen.c3()
    dev = _dev()
    run = QueryRun(ws, dev)
    data_h, preds = {}, {}
    for t in ws.tables:
        dd = datagen.generate_table(ws, t.name, dev)
        data_h[t.name] = {k: v.cpu().numpy() for k, v in dd.items()}
        preds[t.name] = datagen.resolve_preds(ws, t.name)
        run.build_table(t.name, dd, preds[t.name])
        del dd
    torch.cuda.synchronize()
    vec, surv = {}, {}
    for t in ws.tables:
        mask, cnt = oracle.filter_mask(data_h[t.name], preds[t.name])
        surv[t.name] = cnt
        for s in ws.sketches_of(t.name):
            vec[(t.name, s.edge_ids[0])] = oracle.build([data_h[t.name][k] for k in s.key_cols], mask, s.d, s.w,
                                                        s.edge_ids, master=ws.master_seed)
    og = oracle.Graph(surv, ws.edges, vec)
    assert run.survivors.tolist() == [surv[t.name] for t in ws.tables]
    for s, sk in zip(ws.sketches, run.sketches):
        assert np.array_equal(sk.counters.cpu().numpy(), og.vec[(s.table, s.edge_ids[0])]), (s.table, s.edge_ids)
    jg = run.graph()
    subs = oracle.connected_subplans(og)
    assert len(subs) == 14
    for s in subs:
        assert jg.estimate_join_exact(s)[0] == oracle.estimate_rows(og, s, rows=[0])[0], s


# ------------------------------------------------------------------ lookup-table scan (FAST)
def _fast_cols(n, seed, skew):
    rng = np.random.default_rng(seed)
    if skew == "flat":
        a = rng.integers(0, 1 << 20, n)
        b = rng.integers(0, 1 << 20, n)
    else:                                   # Zipf 2.0-like: most lanes of a warp share a key
        a = rng.zipf(2.0, n) % (1 << 20)
        b = rng.zipf(1.3, n) % (1 << 20)
    a = a.astype(np.int32)
    b = b.astype(np.int32)
    if n > 64:                              # keys outside the hinted domain: fallback hashing
        a[::53] = -rng.integers(1, 1 << 30, a[::53].shape[0])
        b[::59] = (1 << 20) + rng.integers(0, 1 << 30, b[::59].shape[0])
        a[:4] = [-1, 7, -(1 << 31), (1 << 31) - 1]   # -1 and 7 share a canonical key (H1)
    return {"a": a, "b": b, "p": rng.integers(0, 1000, n).astype(np.int32)}


FAST_TARGETS = [  # one hash family per key column (edge), matrices on the same families
    (["a"], 5, [1024], ["T1.b|T2.a"]),
    (["b"], 5, [1024], ["T2.b|T3.a"]),
    (["a", "b"], 5, [512, 512], ["T1.b|T2.a", "T2.b|T3.a"]),
    (["a"], 5, [256], ["T1.b|T2.a"]),        # narrower sketch of the same family
]


@pytest.mark.parametrize("n", [1, 4097, 1_000_003])
@pytest.mark.parametrize("skew", ["flat", "zipf"])
@pytest.mark.parametrize("preds", [[], [("p", pb.RANGE, 0, 499)], [("p", pb.RANGE, 0, 9), ("a", pb.RANGE, -(1 << 31), 1 << 19)]])
@pytest.mark.parametrize("fast", ["1", "0"])
def test_lookup_table_scan_equals_oracle(n, skew, preds, fast, capfd, monkeypatch):
    """int32 keys with domain hints (C5 / C2 shape): the lookup-table scan (and, as a second
    witness, the hashing scan with COMPASS_FAST=0) against the oracle, bit for bit."""
    monkeypatch.setenv("COMPASS_FAST", fast)
    monkeypatch.setenv("COMPASS_SCAN_DEBUG", "1")
    cols = _fast_cols(n, 9000 + n, skew)
    g, gs = _build(cols, preds, FAST_TARGETS, domains={"a": 1 << 20, "b": 1 << 20})
    err = capfd.readouterr().err
    if fast == "1":
        assert "fast 1" in err, err
    o, os_ = _oracle(cols, preds, FAST_TARGETS)
    assert gs == os_
    for t, (x, y) in enumerate(zip(g, o)):
        assert np.array_equal(x, y), f"target {t} differs"


def test_wire_pack_unpack_roundtrip_and_overflow_flag():
    """sketch_wire_pack / sketch_wire_unpack (int32 wire format of the merge, SURVEY §8(e) i)."""
    rng = np.random.default_rng(1)
    v = rng.integers(-(1 << 31), 1 << 31, 100_003, dtype=np.int64)
    src = torch.from_numpy(v).to(_dev())
    wire = torch.empty(v.size, dtype=torch.int32, device=_dev())
    flag = torch.zeros(1, dtype=torch.int32, device=_dev())
    pb.sketch_wire_pack(src, wire, flag)
    back = torch.empty_like(src)
    pb.sketch_wire_unpack(wire, back)
    torch.cuda.synchronize()
    assert torch.equal(back, src) and int(flag.item()) == 0
    src[7] = 1 << 31                      # outside int32
    pb.sketch_wire_pack(src, wire, flag)
    torch.cuda.synchronize()
    assert int(flag.item()) == 1


# ------------------------------------------------------------------ §8(f) 3: 3-D partitioned tensors
T3_TARGETS = [  # (key cols, d, w, edge ids in canonical order)
    (["x", "y", "z"], 5, [16, 8, 32], ["A.x|C.x", "B.y|C.y", "C.z|D.z"]),
    (["x"], 5, [256], ["A.x|C.x"]),
    (["y", "y", "x"], 3, [4, 4, 64], ["A.y|C.y", "B.y|C.y", "C.x|E.x"]),   # one column on two dims
]


@pytest.mark.parametrize("n", [1, 4097, 300_001])
@pytest.mark.parametrize("preds", [[], [("p", pb.RANGE, 10, 60)]])
def test_tensor3_build_equals_oracle(n, preds):
    """3-D partitioned tensor sketches built by sketch_update_filtered next to a
    1-D sketch in one scan: counters bit-exact against the oracle's tuple-by-tuple build."""
    rng = np.random.default_rng(n)
    cols = {"x": rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64), "y": rng.zipf(1.3, n).astype(np.int32),
            "z": rng.integers(0, 1000, n).astype(np.int64), "p": rng.integers(0, 100, n).astype(np.int32)}
    g, gs = _build(cols, preds, T3_TARGETS)
    o, os_ = _oracle(cols, preds, T3_TARGETS)
    assert gs == os_
    for a, b in zip(g, o):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("n", [4097, 1_000_003])
@pytest.mark.parametrize("mode", ["scan", "scan_lut", "generic"])
def test_tensor3_scan_paths_equal_oracle(n, mode, capfd, monkeypatch):
    """3-D tensors inside the persistent scan (k_scan drain: hashing, or the per-dimension
    lookup tables when every key column has a domain hint) and in the grid-stride kernel:
    bit-exact counters next to a 1-D sketch and a matrix, keys partly outside the hints."""
    monkeypatch.setenv("COMPASS_SCAN_DEBUG", "1")
    if mode == "generic":
        monkeypatch.setenv("COMPASS_SCAN", "generic")
    rng = np.random.default_rng(n + len(mode))
    a = (rng.zipf(1.3, n) % 3000).astype(np.int32)
    b = rng.integers(0, 5000, n).astype(np.int32)
    a[::89] = 3000 + rng.integers(0, 10**6, a[::89].shape[0]).astype(np.int32)   # above the hint
    cols = {"a": a, "b": b, "p": rng.integers(0, 100, n).astype(np.int32)}
    targets = [(["a", "a", "b"], 7, [64, 16, 32], ["C.a|E.a", "C.a|G.a", "C.b|F.b"]),
               (["a", "b"], 7, [64, 64], ["C.a|E.a", "C.b|F.b"]),
               (["a"], 7, [1024], ["C.a|E.a"])]
    preds = [("p", pb.RANGE, 10, 70)]
    dom = {"a": 3000, "b": 5000} if mode == "scan_lut" else None
    g, gs = _build(cols, preds, targets, domains=dom)
    err = capfd.readouterr().err
    if mode == "generic":
        assert "k_scan plan" not in err
    else:
        assert "k_scan plan: keys 2 preds 1" in err, err
    o, os_ = _oracle(cols, preds, targets)
    assert gs == os_
    for t, (x, y) in enumerate(zip(g, o)):
        assert np.array_equal(x, y), f"target {t} differs"


def _t3_star_graph(rng, d, wv, wt, vmax):
    """centre C with a 3-D tensor over (A.x|C.x, B.y|C.y, C.z|D.z) and leaf vectors; returns
    (oracle graph, JoinGraph)."""
    es = ["A.x|C.x", "B.y|C.y", "C.z|D.z"]
    names = ["A", "B", "C", "D"]
    vec = {("A", es[0]): rng.integers(-vmax, vmax + 1, (d, wv)), ("B", es[1]): rng.integers(-vmax, vmax + 1, (d, wv)),
           ("D", es[2]): rng.integers(-vmax, vmax + 1, (d, wv))}
    for e in es:
        vec[("C", e)] = rng.integers(-vmax, vmax + 1, (d, wv))
    vec = {k: v.astype(np.int64) for k, v in vec.items()}
    ten = rng.integers(-vmax, vmax + 1, (d, wt, wt, wt)).astype(np.int64)
    edges = [(es[0], "A", "C"), (es[1], "B", "C"), (es[2], "C", "D")]
    surv = {t: int(rng.integers(1, 100)) for t in names}
    og = oracle.Graph(surv, edges, vec, {("C", tuple(es)): ten})
    sk = {k: pb.Sketch(d, [wv], [k[1]], 42, _dev(), counters=torch.from_numpy(v).to(_dev())) for k, v in vec.items()}
    tsk = pb.Sketch(d, [wt] * 3, es, 42, _dev(), counters=torch.from_numpy(ten).to(_dev()))
    jedges = [(names.index(u), names.index(v), sk[(u, e)], sk[(v, e)]) for e, u, v in edges]
    jg = pb.JoinGraph(names, [surv[t] for t in names], jedges, [(2, 0, 1, tsk)])
    return og, jg


@pytest.mark.parametrize("vmax", [3, 1 << 20])
def test_tensor3_estimates_equal_oracle(vmax):
    """Sub-plans through a 3-D tensor node (the star centre with all three edges, vectors folded
    to the tensor width) and without it (merged views): exact per row, plans identical."""
    rng = np.random.default_rng(vmax)
    og, jg = _t3_star_graph(rng, 5, 64, 16, vmax)
    for s in oracle.connected_subplans(og):
        assert jg.estimate_join_exact(s) == oracle.estimate_rows(og, s), s
    assert tuple(jg.plan_greedy()) == tuple(oracle.plan_greedy(og))


def test_c3t_scaled_all_subplans_and_plan():
    """C3 with 3-D tensors for MK and CI and a matrix for T (datagen.c3t): the generalised
    partitioned estimator on the paper's running-example shape; counters and
    all 14 sub-plans exact, greedy plan identical."""
    ws = datagen.c3t(scale=0.005, w=256, wt=16)
    dev = _dev()
    run = QueryRun(ws, dev)
    data_h, preds = {}, {}
    for t in ws.tables:
        dd = datagen.generate_table(ws, t.name, dev)
        data_h[t.name] = {k: v.cpu().numpy() for k, v in dd.items()}
        preds[t.name] = datagen.resolve_preds(ws, t.name)
        run.build_table(t.name, dd, preds[t.name])
    torch.cuda.synchronize()
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
    og = oracle.Graph(surv, ws.edges, vec, mat)
    for s, sk in zip(ws.sketches, run.sketches):
        want = vec[(s.table, s.edge_ids[0])] if len(s.w) == 1 else mat[(s.table, tuple(s.edge_ids))]
        assert np.array_equal(sk.counters.cpu().numpy(), want), (s.table, s.edge_ids)
    jg = run.graph()
    for s in oracle.connected_subplans(og):
        assert jg.estimate_join_exact(s) == oracle.estimate_rows(og, s), s
    assert tuple(jg.plan_greedy()) == tuple(oracle.plan_greedy(og))


# ------------------------------------------------------------------ tensor-core modular GEMM (cycles)
def _matrix_ring(rng, T, w, d, vmax):
    """ring of T tables, every table a w x w matrix over its two edges (the conditioned-cycle
    path batches one modular GEMM per interior matrix over the w buckets of the cut edge)."""
    names = [f"t{i}" for i in range(T)]
    eids = [f"{names[i]}.c|{names[(i + 1) % T]}.c" if i + 1 < T else f"{names[0]}.c{i}|{names[i]}.c{i}" for i in range(T)]
    topo = [(i, (i + 1) % T) for i in range(T)]
    vec_np, mat_np = {}, {}
    for i, (u, v) in enumerate(topo):
        for t in (u, v):
            vec_np[(names[t], eids[i])] = rng.integers(-vmax, vmax + 1, (d, w)).astype(np.int64)
    for t in range(T):
        inc = sorted(eids[i] for i, e in enumerate(topo) if t in e)
        mat_np[(names[t], tuple(inc))] = rng.integers(-vmax, vmax + 1, (d, w, w)).astype(np.int64)
    og = oracle.Graph({n: int(rng.integers(1, 1000)) for n in names}, [(eids[i], names[u], names[v]) for i, (u, v) in enumerate(topo)],
                      vec_np, mat_np)
    sk = {}
    for key, arr in vec_np.items():
        s = pb.Sketch(d, [w], [key[1]], 42, _dev(), counters=torch.from_numpy(arr).to(_dev()))
        sk[key] = s
    mats = []
    for (t, inc), arr in mat_np.items():
        s = pb.Sketch(d, [w, w], list(inc), 42, _dev(), counters=torch.from_numpy(arr).to(_dev()))
        mats.append((names.index(t), eids.index(inc[0]), eids.index(inc[1]), s))
    edges = [(u, v, sk[(names[u], eids[i])], sk[(names[v], eids[i])]) for i, (u, v) in enumerate(topo)]
    return og, pb.JoinGraph(names, [og.tables[n] for n in names], edges, mats), names


@pytest.mark.parametrize("T,w,vmax", [(4, 16, 3), (5, 32, 1 << 20), (4, 64, 1 << 40)])
@pytest.mark.parametrize("feed", ["bulk", "tc"])
def test_cycle_gemm_tensor_cores_equal_oracle(T, w, vmax, feed, capfd, monkeypatch):
    """Matrix rings (every table a matrix): the conditioned-cycle estimate runs the modular
    GEMM on tcgen05 (kind::i8 byte planes; fed by bulk copies of pre-tiled planes, or by
    register stores); every row equals the oracle's exact value."""
    monkeypatch.setenv("COMPASS_EST_DEBUG", "1")
    if feed == "tc":
        monkeypatch.setenv("COMPASS_GEMM", "tc")
    rng = np.random.default_rng(T * 1000 + w)
    og, jg, names = _matrix_ring(rng, T, w, 3, vmax)
    full = tuple(names)
    got = jg.estimate_join_exact(full)
    assert ("gemm tc bulk:" if feed == "bulk" else "gemm tc:") in capfd.readouterr().err
    assert got == oracle.estimate_rows(og, full)


@pytest.mark.parametrize("T,w", [(4, 128), (6, 256), (4, 512)])
@pytest.mark.parametrize("feed", ["bulk", "tc"])
def test_cycle_gemm_tensor_cores_equal_cuda_cores(T, w, feed, capfd, monkeypatch):
    """Full-size tiles and several tiles per GEMM (w = 128..512): the tensor-core GEMMs and the
    CUDA-core GEMM give identical exact estimates on every row of every cyclic sub-plan."""
    rng = np.random.default_rng(T * 7 + w)
    og, jg, names = _matrix_ring(rng, T, w, 5, 1 << 30)
    full = tuple(names)
    monkeypatch.setenv("COMPASS_EST_DEBUG", "1")
    if feed == "tc":
        monkeypatch.setenv("COMPASS_GEMM", "tc")
    tc = jg.estimate_join_exact(full)
    assert ("gemm tc bulk:" if feed == "bulk" else "gemm tc:") in capfd.readouterr().err
    monkeypatch.setenv("COMPASS_GEMM", "cuda")
    og2, jg2, _ = _matrix_ring(np.random.default_rng(T * 7 + w), T, w, 5, 1 << 30)
    assert jg2.estimate_join_exact(full) == tc


# ------------------------------------------------------------------ row-sharded composition on the device (§8(e) iii)
@pytest.mark.parametrize("cycle", [False, True])
def test_row_shard_estimates_and_plan_on_device(cycle):
    """The row-shard sketches of rowshard.pack_rows (as 2 and 3 ranks would receive them
    after the reduce-scatter) evaluated by the library's exact estimator: the rows of every
    connected sub-plan concatenate to the full sketches' rows, and merge_rows +
    plan_greedy_rowshard (one process) give plan_greedy's plan."""
    from paper_2102_02440_b200 import rowshard as rs
    ws = datagen.c5(scale=2e-4, cycle=cycle, w=128, wm=64)
    dev = _dev()
    run = QueryRun(ws, dev)
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    run.build(data, preds)
    torch.cuda.synchronize()
    full = run.graph()
    d = ws.sketches[0].d
    adj = {t.name: set() for t in ws.tables}
    for _, u, v in ws.edges:
        adj[u].add(v)
        adj[v].add(u)
    subs, frontier = set(), {(t.name,) for t in ws.tables}
    while frontier:   # connected sub-plans, grown one neighbour at a time
        subs |= frontier
        frontier = {tuple(sorted(S + (x,))) for S in frontier for a in S for x in adj[a] if x not in S} - subs
    want = {S: full.estimate_join_exact(S) for S in subs if len(S) > 1}
    counters = [sk.counters for sk in run.sketches]
    for world in (2, 3):
        send = rs.pack_rows(counters, d, world)
        clen = send.numel() // world
        R = rs.shard_rows(d, world)
        cells = [c[0].numel() for c in counters]
        _, offs = rs.chunk_layout(cells, R)
        got = {S: [] for S in want}
        for rank, (r0, r1) in enumerate(rs.row_ranges(d, world)):
            chunk = send[rank * clen:(rank + 1) * clen]
            shards = [pb.Sketch(R, s.w, s.edge_ids, ws.master_seed, dev, counters=chunk[o:o + R * n].view(R, *s.w))
                      for s, o, n in zip(ws.sketches, offs, cells)]
            g = run.graph(sketches=shards)
            for S in want:
                got[S] += g.estimate_join_exact(S)[:r1 - r0]
        assert got == want, world
    shards, own = run.merge_rows()
    order, pre, cost = run.plan_greedy_rowshard(shards, own)
    o2, p2, c2 = full.plan_greedy()
    assert (tuple(order), pre, cost) == (tuple(o2), p2, c2)
