"""Full-size checks (BASELINE.json sizes, the launch configuration bench.py times).

The oracle cannot replay 10^9-row builds in a test, so at full size the CUDA path is checked
through properties that hold at any size and through independent device paths:
  * linearity: the table built in 8 row shards == built in one call, bit-exact;
  * the same builds with the merge over peer memory fused into every scan == the plain builds;
  * the persistent scan == the grid-stride kernel (`COMPASS_SCAN=generic`, a separate
    implementation of filter + update) counter for counter;
  * survivor counts == a plain torch evaluation of the predicates;
  * estimates: the default engine (int128 dot products, exact int128 contraction after the
    absolute-value bound) == the CRT engine alone, per row, on every connected sub-plan, and the
    greedy / Algorithm 1 plans agree.
"""
import numpy as np
import pytest
import torch

import datagen
from paper_2102_02440_b200.query import QueryRun

pytestmark = pytest.mark.gpu


def _torch_survivors(cols, preds):
    n = next(iter(cols.values())).shape[0]
    m = torch.ones(n, dtype=torch.bool, device=next(iter(cols.values())).device)
    for (c, kind, lo, hi, st) in preds:
        v = cols[c].to(torch.int64)
        if kind == datagen.POINT:
            m &= v == lo
        elif kind == datagen.RANGE:
            m &= (v >= lo) & (v <= hi)
        else:
            s = torch.tensor(sorted(st or []), dtype=torch.int64, device=v.device)
            m &= torch.isin(v, s) if len(s) else torch.zeros_like(m)
    return int(m.sum().item())


def _build(ws, data, preds, dev, shards=1):
    run = QueryRun(ws, dev)
    for t in ws.tables:
        n = t.n_rows
        cuts = np.linspace(0, n, shards + 1).astype(np.int64)
        for a, b in zip(cuts[:-1], cuts[1:]):
            run.build_table(t.name, {c: v[a:b] for c, v in data[t.name].items()}, preds[t.name])
    torch.cuda.synchronize()
    return run


def _counters(run):
    return [sk.counters.clone() for sk in run.sketches], run.survivors.clone()


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_build_linearity_and_independent_kernel(name, monkeypatch):
    dev = torch.device("cuda", 0)
    ws = datagen.c4() if name == "C4" else datagen.c5()
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    one, s1 = _counters(_build(ws, data, preds, dev))
    eight, s8 = _counters(_build(ws, data, preds, dev, shards=8))
    assert torch.equal(s1, s8) and all(torch.equal(a, b) for a, b in zip(one, eight))
    assert s1.tolist() == [_torch_survivors(data[t.name], preds[t.name]) for t in ws.tables]
    # the timed launch configuration with the merge over peer memory fused into each scan
    # (bench.py --merge peer; one rank: the merged buffer is the rank's own)
    peer = QueryRun(ws, dev, merge="peer")
    peer.zero_()
    for t in ws.tables:
        peer.build_table(t.name, data[t.name], preds[t.name])
    peer.allreduce()
    torch.cuda.synchronize()
    pc, ps = _counters(peer)
    assert torch.equal(s1, ps) and all(torch.equal(a, b) for a, b in zip(one, pc))
    peer.close()
    monkeypatch.setenv("COMPASS_SCAN", "generic")
    gen, sg = _counters(_build(ws, data, preds, dev))
    assert torch.equal(s1, sg)
    for s, a, b in zip(ws.sketches, one, gen):
        assert torch.equal(a, b), (s.table, s.edge_ids)


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_size_estimates_engines_agree_and_plans(name, monkeypatch):
    dev = torch.device("cuda", 0)
    ws = datagen.c3() if name == "C3" else datagen.c5()
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    run = _build(ws, data, preds, dev)
    g = run.graph()
    names = g.tables
    adj = {n: set() for n in names}
    for u, v, *_ in [(names[e[0]], names[e[1]]) for e in g._keep[0]]:
        adj[u].add(v)
        adj[v].add(u)
    from itertools import combinations
    subs = []
    for k in range(2, len(names) + 1):
        for c in combinations(names, k):
            seen, st = {c[0]}, [c[0]]
            while st:
                x = st.pop()
                for y in adj[x]:
                    if y in c and y not in seen:
                        seen.add(y)
                        st.append(y)
            if seen == set(c):
                subs.append(c)
    default = {s: g.estimate_join_exact(s) for s in subs}
    greedy, enum = g.plan_greedy(), g.plan_enumerate(mode="limit", max_plans=10)
    monkeypatch.setenv("COMPASS_EST_CRT_ONLY", "1")
    crt = {s: g.estimate_join_exact(s) for s in subs}
    assert default == crt
    assert g.plan_greedy() == greedy
    assert g.plan_enumerate(mode="limit", max_plans=10) == enum
