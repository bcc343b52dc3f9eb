"""CPU-side checks of the boundary: the C-ABI library builds, loads without a GPU,
and exports every symbol include/compass_b200.h declares; host logic that needs no
device (sharding, workload recipes) behaves.  No compute call is made here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "compass_b200.h")).read()
    return sorted(set(re.findall(r"^SK_API\s+[\w\s\*]+?\b(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    syms = _declared_symbols()
    for name in ["sketch_create", "sketch_update_filtered", "sketch_merge", "estimate_join"]:
        assert name in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2102_02440_b200 import _build
    _build.build()
    import paper_2102_02440_b200 as pb
    L = pb.lib()
    syms = _declared_symbols()
    assert sorted(pb.EXPORTS) == syms
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.sk_version()


def test_library_is_sm100a_only():
    import subprocess
    from paper_2102_02440_b200 import _build
    lib = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ["sm_90", "sm_80", "sm_103"]:
        assert other not in out


def test_no_oracle_on_product_path():
    """The product package never imports or links the oracle (DESIGN.md boundary)."""
    pkg = os.path.join(ROOT, "paper_2102_02440_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def test_no_cuda_device_means_error_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2102_02440_b200 as pb
    L = pb.lib()
    desc = pb.sk_desc()
    desc.d, desc.ndim, desc.w[0], desc.master_seed = 5, 1, 1024, 42
    desc.edge_id[0] = b"a.x|b.x"
    h = ctypes.c_void_p()
    st = L.sketch_create(ctypes.byref(desc), 0, None, ctypes.byref(h))
    assert st == pb.SK_ECUDA
    assert b"CUDA" in L.sk_last_error()


def test_shard_ranges_cover_rows_exactly():
    import datagen
    for n in [0, 1, 7, 100, 10**9 + 3]:
        for world in [1, 2, 3, 8]:
            rs = [datagen.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_generator_is_shard_invariant_and_seeded():
    import torch
    import datagen
    ws = datagen.c2(scale=1e-4)
    full = datagen.generate_table(ws, "B")
    parts = [datagen.generate_table(ws, "B", rank=r, world=3) for r in range(3)]
    for c in full:
        assert torch.equal(full[c], torch.cat([p[c] for p in parts]))
    again = datagen.generate_table(ws, "B")
    assert all(torch.equal(full[c], again[c]) for c in full)


def test_workload_shapes_match_baseline_configs():
    import datagen
    c1, c2, c3, c4 = datagen.c1(), datagen.c2(), datagen.c3(), datagen.c4()
    assert [t.n_rows for t in c1.tables] == [100_000, 100_000]
    assert sum(t.n_rows for t in c2.tables) == 30_000_000
    assert sorted(t.n_rows for t in c3.tables) == sorted([2_500_000, 4_500_000, 36_000_000, 134_000, 4_100_000])
    assert c4.tables[0].n_rows == 10**9 and all(s.d == 9 and s.w == [16384] for s in c4.sketches)
    chain, cyc = datagen.c5(), datagen.c5(cycle=True)
    assert len(chain.edges) == 9 and len(cyc.edges) == 10
    assert sum(1 for s in chain.sketches if len(s.w) == 2) == 8
    assert sum(1 for s in cyc.sketches if len(s.w) == 2) == 10
    # C3 canonical edge order quoted in SURVEY.md O11: e4 < e3 < e5 < e1 < e2
    ids = [e[0] for e in c3.edges]
    assert sorted(ids) == ["CI.mid|MK.mid", "CI.mid|T.id", "CI.pid|N.id", "K.id|MK.kid", "MK.mid|T.id"]


def test_crt_moduli_are_distinct_primes_below_2_26():
    """The exact-estimate engine's CRT moduli (csrc/estimate.cu kPrimes): distinct primes
    < 2^26 (so residue products accumulate exactly in 64 bits), >= 700 bits in total."""
    import math
    src = open(os.path.join(ROOT, "paper_2102_02440_b200", "csrc", "estimate.cu")).read()
    body = src[src.index("kPrimes[kMaxMod] = {") + len("kPrimes[kMaxMod] = {"):]
    primes = [int(x) for x in body[:body.index("}")].replace("\n", " ").split(",")]

    def is_prime(n):
        if n < 2:
            return False
        for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
            if n % p == 0:
                return n == p
        d, s = n - 1, 0
        while d % 2 == 0:
            d //= 2
            s += 1
        for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
            x = pow(a, d, n)
            if x in (1, n - 1):
                continue
            for _ in range(s - 1):
                x = x * x % n
                if x == n - 1:
                    break
            else:
                return False
        return True

    assert len(set(primes)) == len(primes) == 28
    assert all(is_prime(p) and p < (1 << 26) for p in primes)
    assert sum(math.log2(p) for p in primes) > 700


def test_plan_enumerate_host_validation_without_device():
    """Algorithm 1's argument checks and a single-table graph run on the host only."""
    import paper_2102_02440_b200 as pb
    L = pb.lib()
    surv = (ctypes.c_int64 * 1)(42)
    g = pb.sk_graph()
    g.n_tables, g.survivors, g.n_edges, g.n_mats = 1, surv, 0, 0
    order = (ctypes.c_uint32 * 1)()
    pre = (ctypes.c_double * 1)()
    cost = ctypes.c_double()
    st = pb.sk_enum_stats()
    cfg = pb.sk_enum_config(0.5, 0.5, pb.ENUM_LIMIT, 10, 0)
    assert L.plan_enumerate(ctypes.byref(g), None, order, pre, ctypes.byref(cost), None, None) == pb.SK_EINVAL
    bad = pb.sk_enum_config(0.5, 0.5, pb.ENUM_LIMIT, 0, 0)
    assert L.plan_enumerate(ctypes.byref(g), ctypes.byref(bad), order, pre, ctypes.byref(cost), None, None) == pb.SK_EINVAL
    bad = pb.sk_enum_config(0.5, 0.5, 9, 1, 0)
    assert L.plan_enumerate(ctypes.byref(g), ctypes.byref(bad), order, pre, ctypes.byref(cost), None, None) == pb.SK_EINVAL
    assert L.plan_enumerate(ctypes.byref(g), ctypes.byref(cfg), order, pre, ctypes.byref(cost), ctypes.byref(st), None) == pb.SK_OK
    assert list(order) == [0] and list(pre) == [42.0] and cost.value == 42.0 and st.plans_completed == 1
