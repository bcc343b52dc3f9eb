"""Multi-rank host logic on CPU (gloo, world_size 2): row shards of every table
(SURVEY.md §8(e)), partial sketches packed in the query's int64 buffer, one SUM
all-reduce -> bit-identical to the single-process build (linearity).
The partial sketches here come from the oracle (no GPU on this host); the GPU path
packs its partials into the same layout (paper_2102_02440_b200.query.QueryRun)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build_packed(ws, rank, world):
    import datagen
    import oracle
    from paper_2102_02440_b200.query import packed_layout
    total, lay = packed_layout(ws)
    buf = torch.zeros(total, dtype=torch.int64)
    names = [t.name for t in ws.tables]
    for ti, t in enumerate(ws.tables):
        cols = {k: v.numpy() for k, v in datagen.generate_table(ws, t.name, "cpu", rank=rank, world=world).items()}
        mask, cnt = oracle.filter_mask(cols, datagen.resolve_preds(ws, t.name))
        buf[ti] += cnt
        for (off, n), s in zip(lay, ws.sketches):
            if s.table != t.name:
                continue
            arr = oracle.build([cols[k] for k in s.key_cols], mask, s.d, s.w, s.edge_ids, master=ws.master_seed)
            buf[off:off + n] += torch.from_numpy(arr.reshape(-1))
    return buf, names


def _worker(rank, world, port, cfg, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    from paper_2102_02440_b200.query import allreduce_packed
    ws = getattr(datagen, cfg[0])(**cfg[1])
    buf, _ = _build_packed(ws, rank, world)
    allreduce_packed(buf)
    if rank == 0:
        torch.save(buf, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [("c1", {"scale": 0.2}), ("c2", {"scale": 2e-4}), ("c5", {"scale": 5e-5, "w": 64, "wm": 32})])
def test_two_rank_allreduce_equals_single_build(cfg, tmp_path):
    import datagen
    world = 2
    out = str(tmp_path / "merged.pt")
    mp.start_processes(_worker, args=(world, _free_port(), cfg, out), nprocs=world, join=True, start_method="spawn")
    merged = torch.load(out)
    ws = getattr(datagen, cfg[0])(**cfg[1])
    single, _ = _build_packed(ws, 0, 1)
    assert torch.equal(merged, single)
    assert int(merged[0]) > 0


def _worker_merge(rank, world, port, cfg, mode, out_path):
    """PackedMerge host logic (per-table asynchronous slices, int32 wire) under gloo: the
    int32 packing kernels are replaced by plain dtype conversions on CPU."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    from paper_2102_02440_b200.query import PackedMerge, table_slices
    ws = getattr(datagen, cfg[0])(**cfg[1])
    buf, _ = _build_packed(ws, rank, world)
    wire, overlap = mode
    m = PackedMerge(buf, len(ws.tables), table_slices(ws), wire, overlap,
                    pack=lambda a, b: b.copy_(a.to(torch.int32)), unpack=lambda a, b: b.copy_(a.to(torch.int64)))
    for t in ws.tables:
        m.reduce_table(t.name)
    m.finish()
    if rank == 0:
        torch.save(buf, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [("i64", True), ("i32", False), ("i32", True)])
def test_two_rank_per_table_and_int32_wire_merge(mode, tmp_path):
    import datagen
    cfg = ("c5", {"scale": 5e-5, "w": 64, "wm": 32})
    world = 2
    out = str(tmp_path / "merged.pt")
    mp.start_processes(_worker_merge, args=(world, _free_port(), cfg, mode, out), nprocs=world, join=True,
                       start_method="spawn")
    merged = torch.load(out)
    ws = getattr(datagen, cfg[0])(**cfg[1])
    single, _ = _build_packed(ws, 0, 1)
    assert torch.equal(merged, single)
