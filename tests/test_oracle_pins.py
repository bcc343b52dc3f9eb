"""Pins of the CPU oracle against what the paper and mathematics fix (SURVEY.md §8(c)
"What pins each part").  CPU only, no GPU.

P1 linearity, P2 injective-hash exactness, P3 unbiasedness, P4 paper worked values,
P5 brute-force contraction, P6 fold identity, P7 hash statistics, P8 filter,
P9 greedy hand traces, P10 C1 estimate vs exact join; plus the exact big-integer
arithmetic against Python ints and published mixer test vectors.
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
from oracle import K_MAT, K_MERGED, K_TEN3, K_VEC, POINT, RANGE, SUBSET

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "paper_pins.json")))
P61 = (1 << 61) - 1


# ---------------------------------------------------------------- P4 / published vectors
def test_mixers_published_vectors():
    L = oracle.lib()
    assert L.or_splitmix64(0) == int(GOLD["splitmix64_first_output_seed0"]["expect"], 16)
    for case in GOLD["fnv1a64"]:
        assert L.or_fnv1a64(case["input"].encode()) == int(case["expect"], 16)


@pytest.mark.parametrize("case", GOLD["merge_minabs"])
def test_merge_rule_paper_values(case):
    """PAPER.md:238, evaluated by the C oracle's merged-tensor path (brute + message passing)."""
    a, b = case["values"]
    tens = [(K_MERGED, [0, 1], [np.array([a]), np.array([b])]),
            (K_VEC, [0], [np.array([1])]), (K_VEC, [1], [np.array([1])])]
    assert oracle.contract_row(tens, [1, 1], brute=True) == case["expect"]
    assert oracle.contract_row(tens, [1, 1]) == case["expect"]
    assert oracle.merge_entry([a, b]) == case["expect"]


def test_merge_tie_keeps_left():
    """ties keep the left (earliest) constituent."""
    tens = [(K_MERGED, [0, 1], [np.array([2]), np.array([-2])]),
            (K_VEC, [0], [np.array([1])]), (K_VEC, [1], [np.array([1])])]
    assert oracle.contract_row(tens, [1, 1], brute=True) == 2


def test_l1_paper_example():
    g = GOLD["l1_permutation"]
    assert oracle.permutation_l1(g["estimates"], g["truths"]) == g["expect"]
    assert oracle.permutation_l1([1, 2, 3], [1, 2, 3]) == 0
    assert oracle.permutation_l1([3, 2, 1], [1, 2, 3]) == 4


@pytest.mark.parametrize("vals,expect", [
    # hand-sorted by eye: [-3, 1, 5, 7, 9] -> 5 (mean 3.8, unsorted middle 7)
    ([9, -3, 7, 1, 5], 5),
    # [-10^25, -4, 0, 2, 3, 8, 10^30] -> 2 (unsorted middle 3; the mean is ~1.4e29)
    ([10**30, -4, 0, 3, -10**25, 8, 2], 2),
    # ties: [1, 2, 2, 2, 3] -> 2
    ([2, 2, 1, 3, 2], 2),
    # all negative, d = 3: [-9, -5, -1] -> -5
    ([-1, -9, -5], -5),
    ([42], 42),
])
def test_median_odd_hand_values(vals, expect):
    """PAPER.md:201 (Fast-AGMS estimate = median over the d rows), d odd (reading R5):
    element (d-1)/2 of the ascending order, checked on hand-sorted unsorted rows where the
    mean and the unsorted middle element both differ from the median."""
    assert oracle.median_odd(vals) == expect


def test_median_odd_rejects_even_d():
    with pytest.raises(AssertionError):
        oracle.median_odd([1, 2])


def test_estimate_is_median_of_rows_hand_example():
    """Two-way estimate of hand-written 5-row sketches (w = 2): per-row dot products by
    hand, then the median."""
    A = np.array([[1, 2], [3, -1], [0, 4], [-2, -2], [5, 0]], dtype=np.int64)
    B = np.array([[2, 1], [1, 1], [1, 1], [3, 1], [1, 7]], dtype=np.int64)
    # rows: 1*2+2*1=4, 3-1=2, 0+4=4, -6-2=-8, 5+0=5  -> sorted [-8, 2, 4, 4, 5] -> 4
    g = oracle.Graph({"A": 10, "B": 10}, [("A.k|B.k", "A", "B")], {("A", "A.k|B.k"): A, ("B", "A.k|B.k"): B})
    est, rows = oracle.estimate(g, ("A", "B"))
    assert rows == [4, 2, 4, -8, 5] and est == 4.0


# ---------------------------------------------------------------- exact arithmetic
def test_bignum_exact_vs_python_int():
    L = oracle.lib()
    rng = random.Random(7)
    import ctypes
    for trial in range(200):
        n = rng.randint(1, 40)
        xs = [rng.choice([rng.randint(-(1 << 63), (1 << 63) - 1), rng.randint(-9, 9), -(1 << 63)]) for _ in range(n)]
        ys = [rng.randint(-(1 << 63), (1 << 63) - 1) for _ in range(n)]
        a = np.array(xs, dtype=np.int64)
        b = np.array(ys, dtype=np.int64)
        buf = ctypes.create_string_buffer(256)
        rc = L.or_bn_selftest_mul_add(n, a.ctypes.data, b.ctypes.data, buf, 256)
        assert rc >= 0
        assert int(buf.value.decode()) == sum(x * y * x for x, y in zip(xs, ys))


def test_bignum_to_double_correctly_rounded():
    L = oracle.lib()
    rng = random.Random(11)
    cases = [[(1 << 53) + 1, 1 << 20], [(1 << 53) + 3, 1 << 30], [-(1 << 53) - 1, 3], [(1 << 62) + 1, (1 << 62) + 1],
             [-(1 << 63), -(1 << 63), -(1 << 63)], [0, 5], [1], [-1], [(1 << 54) - 1]]
    for _ in range(300):
        cases.append([rng.randint(-(1 << 63), (1 << 63) - 1) for _ in range(rng.randint(1, 7))])
    for xs in cases:
        a = np.array(xs, dtype=np.int64)
        prod = 1
        for x in xs:
            prod *= x
        assert L.or_bn_selftest_to_double(len(xs), a.ctypes.data) == float(prod)
        assert L.or_dec_to_double(str(prod).encode()) == float(prod)


def test_field_arithmetic_implementation():
    """Implementation check (not a method pin): mod-p polynomial evaluation vs Python ints."""
    for key in [0, 1, -1, 2**31 - 1, -2**31, 2**63 - 1, -2**63, P61, P61 + 5, 123456789]:
        assert oracle.canon(key) == (key % (1 << 64)) % P61
    for r in range(3):
        e = "A.x|B.y"
        a = [oracle.coef(42, e, r, 0, i) for i in range(4)]
        b = [oracle.coef(42, e, r, 1, i) for i in range(2)]
        assert all(0 <= c < P61 for c in a + b)
        for key in [0, 5, -7, 10**12, 2**40 + 3]:
            x = (key % (1 << 64)) % P61
            v = (((a[3] * x + a[2]) * x + a[1]) * x + a[0]) % P61
            assert oracle.xi(42, e, r, key) == (1 if v & 1 else -1)
            assert oracle.bucket(42, e, r, key, 1024) == ((b[1] * x + b[0]) % P61) % 1024


def test_seed_symmetry_and_distinctness():
    """Both endpoints of an edge see identical seeds; 10^4 (edge,row) pairs have no duplicates."""
    seen = set()
    for e in range(100):
        for r in range(100):
            t = tuple(oracle.coef(42, f"E{e}.a|F{e}.b", r, role, i) for role, n in ((0, 4), (1, 2)) for i in range(n))
            assert t not in seen
            seen.add(t)
    assert oracle.coef(42, "x|y", 3, 0, 1) == oracle.coef(42, "x|y", 3, 0, 1)


# ---------------------------------------------------------------- P7 hash statistics
def test_xi_sign_balance():
    keys = np.arange(100_000, dtype=np.int64)
    sk = oracle.build([keys], None, 9, [1], ["K.id|MK.kid"])      # w = 1 -> row sum = sum_k xi_r(k)
    means = sk[:, 0] / len(keys)
    assert np.all(np.abs(means) < 0.02), means


def test_xi_four_wise_products():
    rng = random.Random(3)
    tuples = []
    while len(tuples) < 200:
        t = rng.sample(range(10**6), 4)
        tuples.append(t)
    tot4 = tot2 = 0
    n = 0
    for s in range(500):
        for (a, b, c, d) in tuples:
            xa, xb, xc, xd = (oracle.xi(1000 + s, "e|f", 0, k) for k in (a, b, c, d))
            tot4 += xa * xb * xc * xd
            tot2 += xa * xb
            n += 1
    assert abs(tot4 / n) < 0.02 and abs(tot2 / n) < 0.02


def test_bucket_chi_square():
    from scipy.stats import chi2
    keys = range(100_000)
    for r in range(2):
        counts = np.zeros(1024, dtype=np.int64)
        for k in keys:
            counts[oracle.bucket(42, "R.key|S.key", r, k, 1024)] += 1
        exp = len(keys) / 1024
        stat = float(((counts - exp) ** 2 / exp).sum())
        assert stat < chi2.ppf(0.999, 1023), stat


# ---------------------------------------------------------------- P8 filter
def test_filter_brute_force_and_prefiltered_build():
    rng = np.random.default_rng(5)
    n = 20_000
    cols = {"a": rng.integers(0, 100, n).astype(np.int32), "b": rng.integers(-50, 50, n).astype(np.int64),
            "c": rng.integers(0, 1000, n).astype(np.int32), "k": rng.integers(0, 500, n).astype(np.int64)}
    S = [3, 7, 999, 500, 11]
    preds = [("a", RANGE, 10, 59), ("b", RANGE, oracle.INT64_MIN, 20), ("c", SUBSET, 0, 0, None)]
    preds[2] = ("c", SUBSET, 0, 0, S + list(range(100, 400)))
    mask, cnt = oracle.filter_mask(cols, preds)
    ref = (cols["a"] >= 10) & (cols["a"] <= 59) & (cols["b"] <= 20) & np.isin(cols["c"], S + list(range(100, 400)))
    assert cnt == int(ref.sum()) and np.array_equal(mask.astype(bool), ref)
    m2, c2 = oracle.filter_mask(cols, [("a", POINT, 42, 42, None)])
    assert c2 == int((cols["a"] == 42).sum())
    m3, c3 = oracle.filter_mask(cols, [])
    assert c3 == n
    m4, c4 = oracle.filter_mask(cols, [("c", SUBSET, 0, 0, [])])
    assert c4 == 0
    sk1 = oracle.build([cols["k"]], mask, 5, [64], ["F.k|G.k"])
    sk2 = oracle.build([cols["k"][ref]], None, 5, [64], ["F.k|G.k"])
    assert np.array_equal(sk1, sk2)
    mk1 = oracle.build([cols["k"], cols["a"]], mask, 3, [16, 32], ["F.k|G.k", "F.a|H.a"])
    mk2 = oracle.build([cols["k"][ref], cols["a"][ref]], None, 3, [16, 32], ["F.k|G.k", "F.a|H.a"])
    assert np.array_equal(mk1, mk2)


# ---------------------------------------------------------------- P1 linearity, P6 fold
def test_linearity_random_shards():
    rng = np.random.default_rng(9)
    for trial in range(30):
        n = int(rng.integers(1, 3000))
        k0 = rng.integers(-10**9, 10**9, n).astype(np.int64)
        k1 = rng.integers(0, 1000, n).astype(np.int32)
        full = oracle.build([k0], None, 3, [128], ["a|b"])
        fullm = oracle.build([k0, k1], None, 3, [16, 8], ["a|b", "c|d"])
        G = int(rng.integers(1, 9))
        cuts = np.sort(rng.integers(0, n + 1, G - 1))
        parts = np.split(np.arange(n), cuts)
        acc = np.zeros_like(full)
        accm = np.zeros_like(fullm)
        for p in parts:
            oracle.build([k0[p]], None, 3, [128], ["a|b"], out=acc)
            oracle.build([k0[p], k1[p]], None, 3, [16, 8], ["a|b", "c|d"], out=accm)
        assert np.array_equal(acc, full) and np.array_equal(accm, fullm)
        # each tuple moves exactly one counter per row by +-1
        assert np.all(np.abs(full).sum(axis=1) <= n) and np.all(full.sum(axis=1) % 2 == n % 2)


def test_fold_identity():
    rng = np.random.default_rng(10)
    for trial in range(10):
        keys = rng.integers(0, 10**6, 5000).astype(np.int32)
        b1024 = oracle.build([keys], None, 5, [1024], ["x|y"])
        for wn in (512, 256, 64):
            assert np.array_equal(oracle.fold(b1024, wn), oracle.build([keys], None, 5, [wn], ["x|y"]))
        k2 = rng.integers(0, 10**6, 5000).astype(np.int32)
        m = oracle.build([keys, k2], None, 3, [64, 32], ["x|y", "z|z2"])
        m2 = oracle.build([keys, k2], None, 3, [16, 8], ["x|y", "z|z2"])
        assert np.array_equal(oracle.fold(oracle.fold(m, 16, axis=1), 8, axis=2), m2)


# ---------------------------------------------------------------- P2 exactness
def _injective_seed(keys, edges_widths, d, start=42):
    s = start
    while True:
        ok = True
        for e, w in edges_widths:
            for r in range(d):
                if len({oracle.bucket(s, e, r, k, w) for k in keys}) != len(keys):
                    ok = False
                    break
            if not ok:
                break
        if ok:
            return s
        s += 1


def test_single_key_exactness():
    """one key, frequencies fA, fB -> every row equals fA*fB."""
    for fa in range(1, 21, 3):
        for fb in range(1, 21, 4):
            A = oracle.build([np.full(fa, 77, dtype=np.int64)], None, 5, [1024], ["A.k|B.k"])
            B = oracle.build([np.full(fb, 77, dtype=np.int32)], None, 5, [1024], ["A.k|B.k"])
            assert all(oracle.two_way_row(A[r], B[r]) == fa * fb for r in range(5))


def test_injective_hash_two_way_and_chain_exact():
    """North-star pin 2 / SURVEY P2: injective h on a tiny domain -> every row exact."""
    rng = np.random.default_rng(12)
    keys = list(range(100, 108))
    e1, e2 = "A.k|B.k", "B.l|C.l"
    d = 3
    seed = _injective_seed(keys, [(e1, 1024), (e1, 64), (e2, 1024), (e2, 64)], d)
    fA = rng.integers(0, 6, 8)
    fC = rng.integers(0, 6, 8)
    fB = rng.integers(0, 4, (8, 8))
    kA = np.repeat(keys, fA).astype(np.int64)
    kC = np.repeat(keys, fC).astype(np.int32)
    pairs = [(keys[i], keys[j]) for i in range(8) for j in range(8) for _ in range(fB[i, j])]
    kB1 = np.array([p[0] for p in pairs], dtype=np.int32)
    kB2 = np.array([p[1] for p in pairs], dtype=np.int64)
    A = oracle.build([kA], None, d, [1024], [e1], master=seed)
    B1 = oracle.build([kB1], None, d, [1024], [e1], master=seed)
    B2 = oracle.build([kB2], None, d, [1024], [e2], master=seed)
    C = oracle.build([kC], None, d, [1024], [e2], master=seed)
    M = oracle.build([kB1, kB2], None, d, [64, 64], [e1, e2], master=seed)
    g = oracle.Graph({"A": len(kA), "B": len(kB1), "C": len(kC)}, [(e1, "A", "B"), (e2, "B", "C")],
                     {("A", e1): A, ("B", e1): B1, ("B", e2): B2, ("C", e2): C}, {("B", (e1, e2)): M})
    ab = oracle.estimate_rows(g, ("A", "B"))
    assert ab == [int((fA * fB.sum(axis=1)).sum())] * d
    abc = oracle.estimate_rows(g, ("A", "B", "C"))
    assert abc == [int(fA @ fB @ fC)] * d
    for r in range(d):   # message passing == literal definition on the chain
        assert oracle.estimate_rows(g, ("A", "B", "C"), brute=False, rows=[r]) == [abc[r]]


# ---------------------------------------------------------------- P3 unbiasedness
def _mean_se(vals):
    v = np.array(vals, dtype=np.float64)
    return v.mean(), v.std(ddof=1) / math.sqrt(len(v))


def test_two_way_unbiased():
    rng = np.random.default_rng(21)
    p = 1.0 / np.arange(1, 13) ** 1.1
    p /= p.sum()
    kA = rng.choice(12, 60, p=p).astype(np.int64)
    kB = rng.choice(12, 60, p=p).astype(np.int64)
    J = int((np.bincount(kA, minlength=12) * np.bincount(kB, minlength=12)).sum())
    ests = []
    for s in range(2000):
        A = oracle.build([kA], None, 1, [4], ["A.k|B.k"], master=5000 + s)
        B = oracle.build([kB], None, 1, [4], ["A.k|B.k"], master=5000 + s)
        ests.append(oracle.two_way_row(A[0], B[0]))
    m, se = _mean_se(ests)
    assert abs(m - J) < 4 * se, (m, J, se)


def test_partitioned_chain_unbiased():
    rng = np.random.default_rng(22)
    kA = rng.integers(0, 6, 40).astype(np.int64)
    kB1 = rng.integers(0, 6, 40).astype(np.int64)
    kB2 = rng.integers(0, 6, 40).astype(np.int64)
    kC = rng.integers(0, 6, 40).astype(np.int64)
    fA, fC = np.bincount(kA, minlength=6), np.bincount(kC, minlength=6)
    fB = np.zeros((6, 6), dtype=np.int64)
    np.add.at(fB, (kB1, kB2), 1)
    J = int(fA @ fB @ fC)
    e1, e2 = "A.k|B.k", "B.l|C.l"
    ests = []
    for s in range(2000):
        A = oracle.build([kA], None, 1, [4], [e1], master=9000 + s)
        C = oracle.build([kC], None, 1, [4], [e2], master=9000 + s)
        M = oracle.build([kB1, kB2], None, 1, [4, 4], [e1, e2], master=9000 + s)
        ests.append(int(A[0] @ M[0] @ C[0]))
    m, se = _mean_se(ests)
    assert abs(m - J) < 4 * se, (m, J, se)


# ---------------------------------------------------------------- P5 contraction vs literal definition
def _random_network(rng, topo, w, vmax=3):
    """topo: list of edges (u, v) over tables 0..T-1 (canonical order = list order)."""
    T = 1 + max(max(e) for e in topo)
    widths = [int(rng.integers(1, w + 1)) for _ in topo]
    tens = []
    for t in range(T):
        inc = [i for i, e in enumerate(topo) if t in e]
        if len(inc) == 1:
            tens.append((K_VEC, inc, [rng.integers(-vmax, vmax + 1, widths[inc[0]])]))
        elif len(inc) == 2 and rng.random() < 0.4:
            tens.append((K_MAT, inc, [rng.integers(-vmax, vmax + 1, widths[inc[0]] * widths[inc[1]])]))
        else:
            tens.append((K_MERGED, inc, [rng.integers(-vmax, vmax + 1, widths[e]) for e in inc]))
    return tens, widths


TOPOLOGIES = [
    [(0, 1)],
    [(0, 1), (1, 2)],
    [(0, 1), (1, 2), (2, 3)],
    [(0, 1), (1, 2), (0, 2)],                          # triangle
    [(0, 1), (1, 2), (2, 0), (2, 3)],                  # triangle + tail
    [(1, 0), (0, 2), (1, 2), (2, 3), (1, 4)],          # C3 shape (triangle 0-1-2, leaves 3, 4)
    [(0, 1), (0, 2), (0, 3)],                          # star: 3-leg merged node
    [(0, 1), (1, 2), (2, 3), (3, 0)],                  # 4-cycle
    [(2, 1), (0, 1), (3, 1), (2, 0)],                  # triangle with 3-leg node + leaf
]


def test_message_passing_equals_literal_definition():
    rng = np.random.default_rng(31)
    for trial in range(400):
        topo = TOPOLOGIES[trial % len(TOPOLOGIES)]
        tens, widths = _random_network(rng, topo, 4)
        assert oracle.contract_row(tens, widths) == oracle.contract_row(tens, widths, brute=True), (trial, topo)


def _c3_graph(rng, w, d=3, vmax=3):
    import datagen
    ws = datagen.c3(scale=1e-4, w=w, d=d)
    vec = {(s.table, s.edge_ids[0]): rng.integers(-vmax, vmax + 1, (d, w)).astype(np.int64) for s in ws.sketches}
    return oracle.Graph({t.name: int(rng.integers(1, 50)) for t in ws.tables}, ws.edges, vec)


def test_c3_subplans_all_14_equal_literal_definition():
    """The C3 recipe with its canonical edge order: every connected sub-plan."""
    rng = np.random.default_rng(41)
    for trial in range(4):
        g = _c3_graph(rng, w=3)
        subs = oracle.connected_subplans(g)
        assert len(subs) == 14
        for s in subs:
            assert oracle.estimate_rows(g, s) == oracle.estimate_rows(g, s, brute=True), s


def test_merged_one_edge_equals_two_way():
    """merged_estimate on one edge == fa_two_way_estimate."""
    rng = np.random.default_rng(42)
    g = _c3_graph(rng, w=64)
    for s in [("K", "MK"), ("CI", "N"), ("MK", "T")]:
        e = g.induced(s)[0][0]
        a, b = s
        assert oracle.estimate_rows(g, s) == [oracle.two_way_row(g.vec[(a, e)][r], g.vec[(b, e)][r]) for r in range(g.d)]


def test_c5_cycle_small_equals_literal():
    import datagen
    rng = np.random.default_rng(43)
    ws = datagen.c5(scale=1e-6, cycle=True, w=4, wm=2, d=1, n_tables=4)
    vec, mat = {}, {}
    for s in ws.sketches:
        if len(s.key_cols) == 1:
            vec[(s.table, s.edge_ids[0])] = rng.integers(-3, 4, (1, 4)).astype(np.int64)
        else:
            mat[(s.table, tuple(s.edge_ids))] = rng.integers(-3, 4, (1, 2, 2)).astype(np.int64)
    g = oracle.Graph({t.name: 5 for t in ws.tables}, ws.edges, vec, mat)
    for s in oracle.connected_subplans(g):
        assert oracle.estimate_rows(g, s) == oracle.estimate_rows(g, s, brute=True), s


# ---------------------------------------------------------------- P9 greedy
class _FakeG(oracle.Graph):
    def __init__(self, tables, edges):
        self.tables, self.edges, self.vec, self.mat, self.d = dict(tables), sorted(edges), {}, {}, 1


def test_greedy_hand_trace():
    g = _FakeG({"a": 10, "b": 100, "c": 5}, [("a.x|b.x", "a", "b"), ("b.y|c.y", "b", "c")])
    est = {("a", "b"): 50.0, ("b", "c"): 20.0, ("a", "b", "c"): 30.0}
    order, prefix, cost = oracle.plan_greedy(g, est_fn=lambda S: est[tuple(sorted(S))])
    assert order == ["c", "b", "a"] and prefix == [5.0, 20.0, 30.0] and cost == 55.0
    # negative estimates are clamped to 0 for planning
    est2 = {("a", "b"): -7.0, ("b", "c"): 20.0, ("a", "b", "c"): 1.0}
    order, prefix, cost = oracle.plan_greedy(g, est_fn=lambda S: est2[tuple(sorted(S))])
    assert order == ["a", "b", "c"] and prefix == [10.0, 0.0, 1.0] and cost == 11.0


def test_greedy_ties_by_alias():
    g = _FakeG({"a": 7, "b": 7, "c": 7}, [("a.x|b.x", "a", "b"), ("b.y|c.y", "b", "c"), ("a.z|c.z", "a", "c")])
    est = {("a", "b"): 3.0, ("b", "c"): 3.0, ("a", "c"): 3.0, ("a", "b", "c"): 1.0}
    order, _, _ = oracle.plan_greedy(g, est_fn=lambda S: est[tuple(sorted(S))])
    assert order == ["a", "b", "c"]


def test_greedy_cost_not_below_exhaustive_minimum():
    """With exact cardinalities, greedy's cost >= min over all valid left-deep orders."""
    import itertools
    rng = np.random.default_rng(51)
    for trial in range(20):
        T = int(rng.integers(3, 6))
        names = [f"t{i}" for i in range(T)]
        edges = [(f"{names[i]}.k|{names[j]}.k", names[i], names[j]) for i in range(1, T) for j in [int(rng.integers(0, i))]]
        card = {}
        g = _FakeG({n: int(rng.integers(1, 100)) for n in names}, edges)

        def est(S):
            S = tuple(sorted(S))
            if S not in card:
                card[S] = float(rng.integers(0, 1000))
            return card[S]
        order, prefix, cost = oracle.plan_greedy(g, est_fn=est)
        best = math.inf
        for perm in itertools.permutations(names):
            ok, c = True, 0.0
            for i in range(1, len(perm) + 1):
                if not oracle.connected(g, perm[:i]):
                    ok = False
                    break
                c += float(g.tables[perm[0]]) if i == 1 else max(est(perm[:i]), 0.0)
            if ok:
                best = min(best, c)
        assert cost >= best


# ---------------------------------------------------------------- Algorithm 1
def _random_graph_cards(rng, T, extra):
    names = [f"t{i}" for i in range(T)]
    edges = [(f"{names[i]}.k|{names[j]}.k", names[i], names[j]) for i in range(1, T) for j in [int(rng.integers(0, i))]]
    for x in range(extra):   # extra edges: cycles and parallel edges (distinct edge ids)
        i, j = sorted(rng.choice(T, 2, replace=False).tolist())
        edges.append((f"{names[i]}.e{x}|{names[j]}.e{x}", names[i], names[j]))
    g = _FakeG({n: int(rng.integers(1, 100)) for n in names}, edges)
    table = {}

    def card_fn(S):   # any non-negative cardinality function (singletons included)
        if S not in table:
            table[S] = float(rng.integers(0, 1000))
        return table[S]
    return g, names, card_fn


def test_enumerate_f_order_hand_example():
    """SPEC.md:363 hand example: cards (8, 8, 64), degrees (1, 2, 1), alpha = beta = 0.5 ->
    f = (0.3125, 0.5625, 0.75): DFS sources v1, v2, v3 in that order."""
    g = _FakeG({"v1": 8, "v2": 8, "v3": 64}, [("v1.a|v2.a", "v1", "v2"), ("v2.b|v3.b", "v2", "v3")])
    seen = []

    def card_fn(S):
        if len(S) == 1 and S[0] not in seen:
            seen.append(S[0])
        return {("v1",): 8, ("v2",): 8, ("v3",): 64}.get(S, 1)
    oracle.plan_enumerate(g, mode="exhaustive", prune=False, card_fn=card_fn)
    assert seen == ["v1", "v2", "v3"]


def test_enumerate_hand_trace_and_prune():
    """3-vertex path a-b-c: from source a (smallest f) the two complete plans
    are found; the source b's first extension exceeds min_cost and is pruned."""
    g = _FakeG({"a": 1, "b": 50, "c": 60}, [("a.x|b.x", "a", "b"), ("b.y|c.y", "b", "c")])
    est = {("a", "b"): 2.0, ("b", "c"): 1000.0, ("a", "b", "c"): 3.0}
    order, pre, cost, st = oracle.plan_enumerate(g, mode="exhaustive", est_fn=lambda S: est[S])
    # a: a(1) -> a,b (2) -> a,b,c (3): cost 6; b: b(50) > 6 -> pruned; c: c(60) > 6 -> pruned
    assert order == ["a", "b", "c"] and pre == [1.0, 2.0, 3.0] and cost == 6.0
    assert st["plans_completed"] == 1 and st["prunes"] == 2


def test_enumerate_exhaustive_is_optimal_and_pruning_sound():
    """with max_plans unbounded the returned cost is the minimum over every
    valid left-deep order (brute force), and disabling pruning changes nothing but the stats;
    without pruning every valid order is completed exactly once."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        g, names, card_fn = _random_graph_cards(rng, int(rng.integers(3, 7)), int(rng.integers(0, 3)))
        costs = oracle.leftdeep_costs_bruteforce(names, g.edges, card_fn)
        o1, p1, c1, s1 = oracle.plan_enumerate(g, mode="exhaustive", card_fn=card_fn)
        o2, p2, c2, s2 = oracle.plan_enumerate(g, mode="exhaustive", prune=False, card_fn=card_fn)
        best = min(costs.values())
        assert c1 == best and c2 == best and costs[tuple(o1)] == best and o1 == o2
        assert s2["plans_completed"] == len(costs) and s2["prunes"] == 0
        assert sum(p1) == c1


def test_enumerate_search_space_nesting():
    """exhaustive <= limit-10 <= full-greedy in cost (same estimator)."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        g, names, card_fn = _random_graph_cards(rng, int(rng.integers(3, 8)), int(rng.integers(0, 4)))
        ce = oracle.plan_enumerate(g, mode="exhaustive", card_fn=card_fn)[2]
        cl = oracle.plan_enumerate(g, mode="limit", max_plans=10, card_fn=card_fn)[2]
        cf = oracle.plan_enumerate(g, mode="full-greedy", card_fn=card_fn)[2]
        c1 = oracle.plan_enumerate(g, mode="limit", max_plans=1, card_fn=card_fn)[2]
        assert ce <= cl <= cf and c1 == cf


# ---------------------------------------------------------------- exact join sizes (accuracy truth)
def _tiny_tables(rng, names, n):
    T = {}
    for t in names:
        cols = {"k": rng.integers(0, 3, n), "j": rng.integers(0, 3, n), "p": rng.integers(0, 10, n)}
        preds = [[], [("p", RANGE, 2, 8)], [("p", SUBSET, 0, 0, [1, 3, 5, 7, 9])], [("p", POINT, 4, 4)]][int(rng.integers(0, 4))]
        T[t] = (cols, preds)
    return T


def test_exact_join_size_equals_nested_loop_definition():
    """Message passing == the literal definition (every combination of one surviving tuple per
    table that agrees on every join edge), on random chains, stars and trees with predicates."""
    rng = np.random.default_rng(21)
    shapes = [[("A", "B", "k", "k")], [("A", "B", "k", "k"), ("B", "C", "j", "j")],
              [("A", "B", "k", "k"), ("A", "C", "j", "k"), ("A", "D", "k", "j")],
              [("A", "B", "k", "j"), ("B", "C", "k", "k"), ("C", "D", "j", "j")]]
    for trial in range(30):
        E = shapes[trial % len(shapes)]
        names = sorted({x for e in E for x in e[:2]})
        T = _tiny_tables(rng, names, int(rng.integers(1, 7)))
        for k in range(1, len(names) + 1):
            for sub in __import__("itertools").combinations(names, k):
                induced = [e for e in E if e[0] in sub and e[1] in sub]
                if len(induced) != len(sub) - 1:
                    continue
                if len(sub) > 1 and not oracle.connected(_FakeG({x: 1 for x in names}, [(f"{u}|{v}", u, v) for u, v, *_ in E]), sub):
                    continue
                assert oracle.exact_join_size(T, E, sub) == oracle.exact_join_size_bruteforce(T, E, sub), (trial, sub)


CYCLIC_SHAPES = [
    # triangle on one shared key column per table (the C3 shape: T.id, MK.mid, CI.mid)
    [("A", "B", "k", "k"), ("A", "C", "k", "k"), ("B", "C", "k", "k")],
    # triangle with a different column per table and edge (a genuine cycle)
    [("A", "B", "k", "j"), ("B", "C", "k", "j"), ("C", "A", "k", "j")],
    # 4-cycle (C5-cycle shape: each table joins on 'k' one way and 'j' the other)
    [("A", "B", "j", "k"), ("B", "C", "j", "k"), ("C", "D", "j", "k"), ("D", "A", "j", "k")],
    # parallel edges between two tables, plus a pendant
    [("A", "B", "k", "k"), ("A", "B", "j", "j"), ("B", "C", "k", "j")],
    # triangle plus two pendants (the C3 graph)
    [("K", "M", "k", "j"), ("M", "T", "k", "k"), ("C", "T", "k", "k"), ("C", "M", "k", "k"), ("C", "N", "j", "k")],
    # trees too (the general routine is not restricted to cycles)
    [("A", "B", "k", "k"), ("B", "C", "j", "j")],
]


def test_exact_join_size_any_equals_nested_loop_definition_with_cycles():
    """exact_join_size_any (hash join with multiplicities) == the literal definition on tiny
    graphs with cycles (one-key and genuine triangles, a 4-cycle, parallel edges, the C3
    graph), every connected sub-plan, random predicates; and == message passing on trees."""
    import itertools
    rng = np.random.default_rng(2102)
    for trial in range(36):
        E = CYCLIC_SHAPES[trial % len(CYCLIC_SHAPES)]
        names = sorted({x for e in E for x in e[:2]})
        T = _tiny_tables(rng, names, int(rng.integers(1, 6)))
        G = _FakeG({x: 1 for x in names}, [(f"{u}.{cu}|{v}.{cv}#{i}", u, v) for i, (u, v, cu, cv) in enumerate(E)])
        for k in range(1, len(names) + 1):
            for sub in itertools.combinations(names, k):
                if len(sub) > 1 and not oracle.connected(G, sub):
                    continue
                want = oracle.exact_join_size_bruteforce(T, E, sub)
                assert oracle.exact_join_size_any(T, E, sub) == want, (trial, sub)
                induced = [e for e in E if e[0] in sub and e[1] in sub]
                if len(induced) == len(sub) - 1:
                    assert oracle.exact_join_size(T, E, sub) == want


def test_exact_join_size_any_hand_triangle():
    """A hand-counted triangle: A(k) = [1, 1, 2], B(k) = [1, 2, 2], C(k) = [1, 2]; all three
    equal on k: key 1 -> 2*1*1 = 2, key 2 -> 1*2*1 = 2, total 4."""
    T = {"A": ({"k": np.array([1, 1, 2])}, []), "B": ({"k": np.array([1, 2, 2])}, []),
         "C": ({"k": np.array([1, 2])}, [])}
    E = [("A", "B", "k", "k"), ("A", "C", "k", "k"), ("B", "C", "k", "k")]
    assert oracle.exact_join_size_any(T, E, ("A", "B", "C")) == 4


def test_accuracy_l1_paper_example():
    """PAPER.md:294 / Table 2: the 4-way joins of JOB 6a, true (6, 1194, 1224) vs sketch
    merging (198, 18M, 6.5M): L1 distance 0 + 1 + 1 = 2, normalised by the 3 sub-plans."""
    truths = {("ci", "k", "mk", "n"): 6, ("ci", "mk", "n", "t"): 1194, ("ci", "k", "mk", "t"): 1224}
    est = {("ci", "k", "mk", "n"): 198, ("ci", "mk", "n", "t"): 18_000_000, ("ci", "k", "mk", "t"): 6_500_000}
    rep = oracle.accuracy_report(est, truths)
    assert rep[4][1] == 2 / 3
    assert rep[4][0] == [198 / 6, 6_500_000 / 1224, 18_000_000 / 1194]


# ---------------------------------------------------------------- P10 C1 end to end
def test_c1_estimate_vs_exact_join():
    import datagen
    ws = datagen.c1()
    R = {k: v.numpy() for k, v in datagen.generate_table(ws, "R").items()}
    S = {k: v.numpy() for k, v in datagen.generate_table(ws, "S").items()}
    mask, nR = oracle.filter_mask(R, datagen.resolve_preds(ws, "R"))
    assert abs(nR / len(mask) - 14 / 125) < 0.01       # attr uniform [1900,2025) > 2010 -> 14/125
    e = ws.edges[0][0]
    A = oracle.build([R["key"]], mask, 5, [1024], [e])
    B = oracle.build([S["key"]], None, 5, [1024], [e])
    fR = np.bincount(R["key"][mask.astype(bool)], minlength=10000)
    fS = np.bincount(S["key"], minlength=10000)
    J = int((fR * fS).sum())
    rows = [oracle.two_way_row(A[r], B[r]) for r in range(5)]
    est = oracle.median_odd(rows)
    sigma = math.sqrt((float((fR ** 2).sum()) * float((fS ** 2).sum()) + J * J) / 1024)
    assert abs(est - J) < 4 * sigma, (est, J, sigma)


# ---------------------------------------------------------------- §8(f) 3: n-D partitioned tensors
def test_tensor3_build_single_tuple_definition():
    """PAPER.md:225 ("a table with 3 joins has a 3-D tensor as its sketch, with one dimension
    for every join attribute"): one tuple (x, y, z) puts exactly prod_q xi^{e_q}_r(x_q) at
    [h^{e_0}_r(x)][h^{e_1}_r(y)][h^{e_2}_r(z)] of every row r and nothing elsewhere; the
    hash primitives are the pinned H3/H4 ones (oracle.xi, oracle.bucket)."""
    es = ["A.x|C.x", "B.y|C.y", "C.z|D.z"]
    w = [8, 4, 16]
    for (x, y, z) in [(5, -3, 1 << 40), (0, 0, 0), (-(1 << 63), (1 << 61) - 1, 7)]:
        T = oracle.build([np.array([x], np.int64), np.array([y], np.int64), np.array([z], np.int64)], None, 3, w, es,
                         master=77)
        for r in range(3):
            want = np.zeros(w, dtype=np.int64)
            idx = tuple(oracle.bucket(77, e, r, k, wq) for e, k, wq in zip(es, (x, y, z), w))
            want[idx] = oracle.xi(77, es[0], r, x) * oracle.xi(77, es[1], r, y) * oracle.xi(77, es[2], r, z)
            assert np.array_equal(T[r], want), (x, y, z, r)


def test_tensor3_linearity_and_fold():
    """P1 and P6 for 3-D tensors: shards sum bit-exactly;
    folding any axis of build(w) equals build at the narrower width."""
    rng = np.random.default_rng(301)
    n = 3000
    keys = [rng.integers(-50, 50, n).astype(np.int64), rng.integers(0, 20, n).astype(np.int32),
            rng.zipf(1.4, n).astype(np.int64)]
    mask = (rng.random(n) < 0.7).astype(np.uint8)
    es = ["A.x|C.x", "B.y|C.y", "C.z|D.z"]
    full = oracle.build(keys, mask, 5, [16, 8, 32], es)
    cuts = sorted(rng.choice(np.arange(1, n), 4, replace=False))
    acc = np.zeros_like(full)
    for a, b in zip([0] + cuts, cuts + [n]):
        acc += oracle.build([k[a:b] for k in keys], mask[a:b], 5, [16, 8, 32], es)
    assert np.array_equal(acc, full)
    narrow = oracle.build(keys, mask, 5, [4, 8, 2], es)
    f = oracle.fold(oracle.fold(full, 4, axis=1), 2, axis=3)
    assert np.array_equal(f, narrow)


def _star3(rng, keys):
    """center C(x, y, z) with leaves A(x), B(y), D(z); random multiplicities on `keys`."""
    k = len(keys)
    fA, fB, fD = rng.integers(0, 4, k), rng.integers(0, 4, k), rng.integers(0, 4, k)
    fC = rng.integers(0, 3, (k, k, k))
    kA = np.repeat(keys, fA).astype(np.int64)
    kB = np.repeat(keys, fB).astype(np.int32)
    kD = np.repeat(keys, fD).astype(np.int64)
    trip = [(keys[i], keys[j], keys[l]) for i in range(k) for j in range(k) for l in range(k) for _ in range(fC[i, j, l])]
    kC = [np.array([t[q] for t in trip], dtype=np.int64) for q in range(3)]
    J = int(np.einsum("i,j,l,ijl->", fA, fB, fD, fC))
    return kA, kB, kD, kC, J


def test_tensor3_star_exact_with_injective_hashes():
    """SURVEY P2 generalised to a 3-D tensor: with every h_r injective on the key domain (at
    the tensor width, and at the vectors' width before folding), every row of the 4-table
    star estimate equals the exact join size sum fA(x) fB(y) fD(z) fC(x, y, z)."""
    rng = np.random.default_rng(302)
    keys = list(range(200, 206))
    es = ["A.x|C.x", "B.y|C.y", "C.z|D.z"]
    d = 3
    seed = _injective_seed(keys, [(e, w) for e in es for w in (256, 16)], d)
    kA, kB, kD, kC, J = _star3(rng, keys)
    vec = {("A", es[0]): oracle.build([kA], None, d, [256], [es[0]], master=seed),
           ("B", es[1]): oracle.build([kB], None, d, [256], [es[1]], master=seed),
           ("D", es[2]): oracle.build([kD], None, d, [256], [es[2]], master=seed)}
    for q, e in enumerate(es):
        vec[("C", e)] = oracle.build([kC[q]], None, d, [256], [e], master=seed)
    T = oracle.build(kC, None, d, [16, 16, 16], es, master=seed)
    g = oracle.Graph({"A": len(kA), "B": len(kB), "C": len(kC[0]), "D": len(kD)},
                     [(es[0], "A", "C"), (es[1], "B", "C"), (es[2], "C", "D")], vec, {("C", tuple(es)): T})
    rows = oracle.estimate_rows(g, ("A", "B", "C", "D"))
    assert rows == [J] * d
    assert oracle.estimate_rows(g, ("A", "B", "C", "D"), brute=True) == rows


def test_tensor3_star_unbiased():
    """SURVEY P3 for the 3-D partitioned estimator ("this procedure can be
    generalized to any number of join attributes"): over 2000 master seeds the mean of the
    per-row estimate is within 4 standard errors of the exact join size."""
    rng = np.random.default_rng(303)
    kA, kB, kD, kC, J = _star3(rng, list(range(5)))
    es = ["A.x|C.x", "B.y|C.y", "C.z|D.z"]
    ests = []
    for s in range(2000):
        A = oracle.build([kA], None, 1, [4], [es[0]], master=20000 + s)[0]
        B = oracle.build([kB], None, 1, [4], [es[1]], master=20000 + s)[0]
        D = oracle.build([kD], None, 1, [4], [es[2]], master=20000 + s)[0]
        T = oracle.build(kC, None, 1, [4, 4, 4], es, master=20000 + s)[0]
        ests.append(int(np.einsum("i,j,l,ijl->", A, B, D, T)))
    m, se = _mean_se(ests)
    assert abs(m - J) < 4 * se, (m, J, se)


def test_tensor3_message_passing_equals_literal_definition():
    """P5 with 3-D tensor nodes: in a star (3 children), at a leaf-bearing tree node, and
    inside a cycle (the conditioned edge fixes one leg) — message passing == definition."""
    rng = np.random.default_rng(304)
    topos = [[(0, 1), (0, 2), (0, 3)],                   # node 0: 3-D star centre
             [(0, 1), (1, 2), (2, 0), (1, 3)],           # node 1: 3-D inside the triangle
             [(1, 0), (0, 2), (1, 2), (2, 3), (1, 4)]]   # C3 shape: nodes 1 and 2 are 3-D
    for trial in range(150):
        topo = topos[trial % len(topos)]
        T = 1 + max(max(e) for e in topo)
        widths = [int(rng.integers(1, 4)) for _ in topo]
        tens = []
        for t in range(T):
            inc = [i for i, e in enumerate(topo) if t in e]
            if len(inc) == 3:
                tens.append((K_TEN3, inc, [rng.integers(-3, 4, widths[inc[0]] * widths[inc[1]] * widths[inc[2]])]))
            elif len(inc) == 2:
                tens.append((K_MAT, inc, [rng.integers(-3, 4, widths[inc[0]] * widths[inc[1]])]))
            else:
                tens.append((K_VEC, inc, [rng.integers(-3, 4, widths[inc[0]])]))
        assert oracle.contract_row(tens, widths) == oracle.contract_row(tens, widths, brute=True), (trial, topo)
