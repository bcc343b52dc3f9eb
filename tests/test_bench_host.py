"""Host logic of bench.py (CPU): sub-plan enumeration, algorithmic bytes, the roof
arithmetic of the bench line, and the multi-threaded oracle baseline's merge."""
import numpy as np
import torch

import bench
import datagen
import oracle


def test_connected_subplan_counts_match_survey():
    """C3 14, C5 chain 45, C5 cycle 81 connected sub-plans (>= 2 tables)."""
    assert len(bench._subplans(datagen.c3(scale=1e-4))) == 14
    assert len(bench._subplans(datagen.c5(scale=1e-6))) == 45
    assert len(bench._subplans(datagen.c5(scale=1e-6, cycle=True))) == 81


def test_algorithmic_bytes_by_hand():
    """SURVEY §8(d) B_alg on C1 at 1 % scale: the predicate column in full, 32-B sectors of the
    key column holding a survivor, the unfiltered table's key column in full, sketch bytes."""
    ws = datagen.c1(scale=0.01)
    data = {t.name: datagen.generate_table(ws, t.name) for t in ws.tables}
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    run = type("R", (), {"sketch_bytes": 2 * 5 * 1024 * 8})()
    got = bench.algorithmic_bytes(ws, data, preds, run)
    n = 1000
    attr = data["R"]["attr"].numpy()
    mask = attr >= 2011
    sectors = sum(1 for i in range(0, n, 8) if mask[i:i + 8].any())
    assert got["alg"] == n * 4 + 32 * sectors + n * 4 + run.sketch_bytes
    assert got["full"] == 3 * n * 4 + run.sketch_bytes


def test_int_update_roofs_arithmetic():
    ws = datagen.c1(scale=0.01)
    roofs = {"hash_narrow_pairs_per_s": 1e11, "hash_wide_pairs_per_s": 5e10, "atoms_smem_per_s": 1e12,
             "red_l2_u64_mat10mb_per_s": 2e11}
    r = bench._int_update_roofs(ws, [100, 1000], 0.001, roofs)   # 1 us of scan time
    pairs = (100 + 1000) * 5          # one (xi, h) pair per survivor and row, int32 keys
    assert r["int"]["hash_pairs"] == pairs and r["update"]["counter_increments"] == pairs
    assert abs(r["int_frac"] - pairs / 1e11 / 1e-6) < 1e-4
    assert abs(r["update_frac"] - pairs / 1e12 / 1e-6) < 1e-4   # 5 x 1024 int32 fits a CTA


def test_threaded_oracle_baseline_merges_private_sketches():
    """cpu_baseline: row ranges built on several threads and merged by int64 addition equal
    the single-threaded build (O4)."""
    ws = datagen.c2(scale=2e-4)
    cols = {t.name: {k: v.numpy() for k, v in datagen.generate_table(ws, t.name).items()} for t in ws.tables}
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    one, four = {}, {}
    bench._oracle_pass(ws, cols, preds, 1, out=one)
    bench._oracle_pass(ws, cols, preds, 4, out=four)
    for t in ws.tables:
        for a, b in zip(one[t.name], four[t.name]):
            assert np.array_equal(a, b)


def test_binding_roof_by_hand():
    """Per-table binding roof: max(HBM, update, hash) per table, summed; lookup-table tables
    (int32 keys with small hinted domains) take no hash term."""
    ws = datagen.c5(scale=1e-6)
    roofs = {"hash_narrow_pairs_per_s": 1e11, "hash_wide_pairs_per_s": 5e10, "atoms_smem_per_s": 1e12,
             "red_l2_u64_mat10mb_per_s": 2e11}
    names = [t.name for t in ws.tables]
    surv = [0] * len(names)
    surv[8] = 10_000_000                          # T9: two 1-D sketches (smem) + one 512^2 matrix (L2)
    per_bytes = {n: 1_000_000_000 for n in names}  # 1 GB each -> 1/6 ms at 6000 GB/s
    r = bench.binding_roof(ws, surv, per_bytes, 10.0, 6000.0, roofs)
    t_hbm = 1e9 / 6e12
    t9 = 2 * 10_000_000 * 5 / 1e12 + 10_000_000 * 5 / 2e11      # 0.1 ms + 0.25 ms
    assert r["per_table"]["T9"]["bound"] == "update"
    assert abs(r["per_table"]["T9"]["roof_ms"] - t9 * 1e3) < 1e-3
    assert r["per_table"]["T1"]["bound"] == "hbm"
    assert abs(r["roof_time_ms"] - (9 * t_hbm + t9) * 1e3) < 1e-3
    assert abs(r["frac"] - r["roof_time_ms"] / 10.0) < 1e-4
