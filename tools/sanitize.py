#!/usr/bin/env python
"""Small builds through every k_scan variant, for compute-sanitizer (memcheck, racecheck,
synccheck; SURVEY.md §4 "Sanitizers", §5 "Race detection"):

    compute-sanitizer --tool racecheck python tools/sanitize.py

Variants: generic KW=0 (int64 range + subset predicates), KW=4 / KW=8 specialised scans,
ring-overflow rounds (100 % selectivity, two key columns), histogram mode with heavy-hitter
tables (hinted key domain), the lookup-table path (int32 keys with hints, matrix + pair
table), sub-tiled stages (very selective predicate), the staged no-predicate path, 3-D
tensors (k_scan drain), and the estimate kernels (two-way, merged views, CRT).
Each build is checked against the oracle so a silent corruption also fails.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2102_02440_b200 as pb  # noqa: E402


def build(cols, preds, targets, domains=None):
    dev = torch.device("cuda", 0)
    names = list(cols)
    dcols = [torch.from_numpy(cols[c]).to(dev) for c in names]
    sks = [pb.Sketch(d, w, e, 42, dev) for (_, d, w, e) in targets]
    surv = torch.zeros(1, dtype=torch.int64, device=dev)
    pr = [(names.index(p[0]),) + tuple(p[1:]) for p in preds]
    tg = [(sk, [names.index(k) for k in t[0]]) for sk, t in zip(sks, targets)]
    dom = [domains.get(c, 0) for c in names] if domains else None
    pb.sketch_update_filtered(dcols, len(cols[names[0]]), pr, tg, survivors=surv, domains=dom)
    torch.cuda.synchronize()
    mask, cnt = oracle.filter_mask(cols, preds)
    assert int(surv.item()) == cnt
    for sk, (keys, d, w, e) in zip(sks, targets):
        assert np.array_equal(sk.counters.cpu().numpy(), oracle.build([cols[k] for k in keys], mask, d, w, e))
    return sks


def main():
    n = 60_000
    rng = np.random.default_rng(5)
    cols = {"k32": rng.integers(-1000, 1000, n).astype(np.int32), "k64": rng.integers(-(1 << 40), 1 << 40, n),
            "z": (rng.zipf(1.5, n) % 3000).astype(np.int32), "a": rng.integers(0, 1 << 16, n).astype(np.int32),
            "p": rng.integers(0, 1000, n).astype(np.int32), "s": rng.integers(0, 50, n).astype(np.int64)}
    T1 = [(["k32"], 5, [1024], ["A.k32|B.x"]), (["k64"], 3, [64], ["A.k64|C.y"])]
    cases = [
        ("generic KW0", [("s", pb.RANGE, 5, 40), ("p", pb.SUBSET, 0, 0, list(range(0, 1000, 7)))], T1, None),
        ("KW4", [("p", pb.RANGE, 0, 499)], [(["k32"], 5, [1024], ["A.k32|B.x"]), (["z"], 3, [64], ["A.z|D.z"])], None),
        ("KW8 + global atomics", [("p", pb.RANGE, 0, 499)], [(["k64"], 9, [16384], ["A.k64|C.y"])], None),
        ("ring overflow", [("p", pb.RANGE, 0, 999)], [(["k32", "k64"], 3, [32, 16], ["A.k32|B.x", "A.k64|C.y"])], None),
        ("histogram + hh", [("p", pb.RANGE, 0, 700)], [(["z"], 5, [1024], [f"A.z|T{i}.z"]) for i in range(10)], {"z": 3000}),
        ("lookup table + pair table", [("p", pb.RANGE, 0, 300)],
         [(["a"], 5, [1024], ["T1.b|T2.a"]), (["z"], 5, [1024], ["T2.b|T3.a"]),
          (["a", "z"], 5, [512, 512], ["T1.b|T2.a", "T2.b|T3.a"])], {"a": 1 << 16, "z": 3000}),
        ("sub-tiled stages", [("p", pb.RANGE, 0, 3)], [(["a"], 5, [1024], ["T1.b|T2.a"])], {"a": 1 << 16, "p": 1000}),
        ("staged keys, no predicate", [], [(["a"], 5, [1024], ["T1.b|T2.a"]), (["k32"], 3, [256], ["A.k32|B.x"])], None),
        ("3-D tensor", [("p", pb.RANGE, 0, 600)], [(["a", "k32", "z"], 3, [8, 8, 16], ["A.a|X.a", "A.k32|Z.k", "A.z|Y.z"])], None),
    ]
    for name, preds, targets, dom in cases:
        build(cols, preds, targets, dom)
        print("ok", name, flush=True)
    # estimates: two-way, merged 3-table view, CRT (matrix chain)
    sks = build(cols, [("p", pb.RANGE, 0, 500)],
                [(["k32"], 3, [64], ["A.k|B.k"]), (["z"], 3, [64], ["B.j|C.j"]), (["k32", "z"], 3, [64, 64], ["A.k|B.k", "B.j|C.j"])])
    g = pb.JoinGraph(["A", "B", "C"], [100, 100, 100], [(0, 1, sks[0], sks[0]), (1, 2, sks[1], sks[1])], [(1, 0, 1, sks[2])])
    g.estimate_join_exact(("A", "B"))
    g.estimate_join_exact(("A", "B", "C"))
    g2 = pb.JoinGraph(["A", "B", "C"], [100, 100, 100], [(0, 1, sks[0], sks[0]), (1, 2, sks[1], sks[1])], [])
    g2.estimate_join_exact(("A", "B", "C"))
    g2.plan_greedy()
    print("ok estimates", flush=True)


if __name__ == "__main__":
    main()
