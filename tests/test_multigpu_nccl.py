"""Multi-GPU path on real devices: N ranks, one GPU each, NCCL
process group; every rank builds its contiguous row shard of every table with the CUDA scan
into the query's packed int64 buffer, then QueryRun.allreduce() merges them (one NCCL SUM).
The merged buffer must equal the oracle's single-process build bit for bit, and every rank
must produce the same greedy plan.  Skipped when fewer than 2 GPUs are visible (the gpurun
pool has one); the same host logic runs on CPU under gloo in tests/test_multirank_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, mode, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    ws = getattr(datagen, cfg[0])(**cfg[1])
    run = QueryRun(ws, dev, wire=mode[0], overlap=mode[1])
    for t in ws.tables:
        data = datagen.generate_table(ws, t.name, dev, rank=rank, world=world)
        run.build_table(t.name, data, datagen.resolve_preds(ws, t.name))
    run.allreduce()
    plan = run.graph().plan_greedy() if ws.kind == "graph" else None
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    if rank == 0:
        torch.save({"buf": run.buffer.cpu(), "plans": plans}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def _oracle_packed(ws):
    import datagen
    import oracle
    from paper_2102_02440_b200.query import packed_layout
    total, lay = packed_layout(ws)
    buf = np.zeros(total, dtype=np.int64)
    for ti, t in enumerate(ws.tables):
        cols = {k: v.numpy() for k, v in datagen.generate_table(ws, t.name, "cpu").items()}
        mask, cnt = oracle.filter_mask(cols, datagen.resolve_preds(ws, t.name))
        buf[ti] = cnt
        for (off, n), s in zip(lay, ws.sketches):
            if s.table == t.name:
                buf[off:off + n] = oracle.build([cols[k] for k in s.key_cols], mask, s.d, s.w, s.edge_ids,
                                                master=ws.master_seed).reshape(-1)
    return buf


@pytest.mark.parametrize("cfg", [("c1", {}), ("c5", {"scale": 2e-4, "w": 128, "wm": 64}),
                                 ("c4", {"scale": 0.002})])
@pytest.mark.parametrize("mode", [("i64", False), ("i32", True)])
def test_nccl_ranks_merge_equals_oracle_build(cfg, mode, tmp_path):
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(world, 8)
    import datagen
    out = str(tmp_path / "merged.pt")
    mp.start_processes(_worker, args=(world, _free_port(), cfg, mode, out), nprocs=world, join=True,
                       start_method="spawn")
    res = torch.load(out)
    ws = getattr(datagen, cfg[0])(**cfg[1])
    assert np.array_equal(res["buf"].numpy(), _oracle_packed(ws))
    assert all(p == res["plans"][0] for p in res["plans"])


def _worker_one(rank, world, port, mode, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    ws = datagen.c5(scale=2e-4, w=128, wm=64)
    run = QueryRun(ws, dev, wire=mode[0], overlap=mode[1], always_merge=True)
    for t in ws.tables:
        run.build_table(t.name, datagen.generate_table(ws, t.name, dev), datagen.resolve_preds(ws, t.name))
    run.allreduce()
    torch.cuda.synchronize()
    torch.save({"buf": run.buffer.cpu()}, out_path)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [("i64", False), ("i32", True)])
def test_nccl_merge_path_on_one_gpu(mode, tmp_path):
    """The merge code path on the device with a one-rank NCCL group (the pool has one GPU):
    per-table int32 packing by the library, NCCL all-reduces on NCCL's stream (asynchronous,
    overlapping the next scan), unpacking — the packed buffer equals the oracle's build."""
    import datagen
    out = str(tmp_path / "one.pt")
    mp.start_processes(_worker_one, args=(1, _free_port(), mode, out), nprocs=1, join=True, start_method="spawn")
    res = torch.load(out)
    assert np.array_equal(res["buf"].numpy(), _oracle_packed(datagen.c5(scale=2e-4, w=128, wm=64)))


def _worker_rows(rank, world, port, cycle, out_path):
    """Row-sharded merge over NCCL (reduce-scatter by sketch row) and the greedy over gathered
    per-row values; on one GPU the group has one rank (the collectives still run)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    gpu = rank if torch.cuda.device_count() > 1 else 0
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    ws = datagen.c5(scale=2e-4, w=128, wm=64, cycle=cycle)
    run = QueryRun(ws, dev)
    for t in ws.tables:
        run.build_table(t.name, datagen.generate_table(ws, t.name, dev, rank=rank, world=world),
                        datagen.resolve_preds(ws, t.name))
    shards, own = run.merge_rows()
    plan = run.plan_greedy_rowshard(shards, own)
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    if rank == 0:
        torch.save({"plans": plans}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cycle", [False, True])
def test_nccl_row_sharded_plan_equals_oracle(cycle, tmp_path):
    """SURVEY.md §8(e) lever iii on NCCL: every rank's plan equals the oracle's greedy plan on
    the single-process build (all visible GPUs, at least a one-rank group)."""
    import datagen
    import oracle
    from paper_2102_02440_b200.query import packed_layout
    world = max(1, min(torch.cuda.device_count(), 8))
    out = str(tmp_path / "rows.pt")
    mp.start_processes(_worker_rows, args=(world, _free_port(), cycle, out), nprocs=world, join=True,
                       start_method="spawn")
    res = torch.load(out)
    ws = datagen.c5(scale=2e-4, w=128, wm=64, cycle=cycle)
    buf = _oracle_packed(ws)
    _, lay = packed_layout(ws)
    vec, mat = {}, {}
    for (o, n), s in zip(lay, ws.sketches):
        arr = buf[o:o + n].reshape(s.d, *s.w)
        if len(s.w) == 1:
            vec[(s.table, s.edge_ids[0])] = arr
        else:
            mat[(s.table, tuple(s.edge_ids))] = arr
    og = oracle.Graph({t.name: int(buf[i]) for i, t in enumerate(ws.tables)}, ws.edges, vec, mat)
    o_order, o_pre, _ = oracle.plan_greedy(og)
    for order, pre, _ in res["plans"]:
        assert tuple(order) == tuple(o_order) and pre == o_pre
