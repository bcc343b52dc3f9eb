"""Cross-GPU merge over peer memory (SURVEY.md §8(f) 4, P2P variant of the fused flush +
all-reduce): every rank pushes its partial sketches into every rank's merged
buffer (CUDA IPC mappings, red.add), fused into the scan's cooperative launch.

The merged buffer must equal the oracle's single-process build bit for bit:
  * one process (the rank's own merged buffer is the only peer) through the fused path
    (k_scan tail) and through the unfused one (generic kernel, then k_peer_push);
  * N ranks: N processes, one GPU each when the box has N GPUs; on the one-GPU pool two
    processes share the GPU — their kernels never wait on each other (the only waits are
    each kernel's own grid barrier and host barriers between complete steps), so this is a
    functional test of the IPC mappings and the pushes, not a stand-in for a scaling run."""
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


CFGS = [("c1", {}), ("c5", {"scale": 2e-4, "w": 128, "wm": 64}), ("c4", {"scale": 0.002}),
        ("c5", {"scale": 2e-4, "w": 128, "wm": 64, "cycle": True})]


@pytest.mark.parametrize("cfg", CFGS)
def test_peer_merge_one_process_fused(cfg):
    """One process: the fused push (k_scan tail after a grid barrier) lands every partial in
    the merged buffer; twice in a row (the merged buffer is zeroed per step)."""
    import datagen
    import paper_2102_02440_b200 as pb
    from paper_2102_02440_b200.query import QueryRun
    dev = torch.device("cuda", 0)
    ws = getattr(datagen, cfg[0])(**cfg[1])
    ref = _oracle_packed(ws)
    run = QueryRun(ws, dev, merge="peer")
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    for _ in range(2):
        run.zero_()
        l0 = pb.kernel_launches()
        for t in ws.tables:
            run.build_table(t.name, data[t.name], datagen.resolve_preds(ws, t.name))
        l1 = pb.kernel_launches()
        run.allreduce()
        torch.cuda.synchronize()
        assert np.array_equal(run.buffer.cpu().numpy(), ref)
        assert np.array_equal(run.merge.final.tensor.cpu().numpy(), ref)
    # fused: the scans launched no separate push kernel (same launch count as a plain build)
    plain = QueryRun(ws, dev)
    for _ in range(2):   # the second build: lookup tables already cached, as in the loop above
        p0 = pb.kernel_launches()
        for t in ws.tables:
            plain.build_table(t.name, data[t.name], datagen.resolve_preds(ws, t.name))
        p1 = pb.kernel_launches()
    torch.cuda.synchronize()
    assert l1 - l0 == p1 - p0
    run.close()
    plain.close()


def test_peer_merge_one_process_unfused(monkeypatch):
    """The grid-stride kernel (COMPASS_SCAN=generic) cannot fuse: one k_peer_push follows each
    scan; same merged buffer."""
    import datagen
    import paper_2102_02440_b200 as pb
    from paper_2102_02440_b200.query import QueryRun
    monkeypatch.setenv("COMPASS_SCAN", "generic")
    dev = torch.device("cuda", 0)
    ws = datagen.c5(scale=2e-4, w=128, wm=64)
    run = QueryRun(ws, dev, merge="peer")
    run.zero_()
    l0 = pb.kernel_launches()
    for t in ws.tables:
        run.build_table(t.name, datagen.generate_table(ws, t.name, dev), datagen.resolve_preds(ws, t.name))
    l1 = pb.kernel_launches()
    run.allreduce()
    torch.cuda.synchronize()
    assert l1 - l0 >= 2 * len(ws.tables)   # scan + push per table
    assert np.array_equal(run.buffer.cpu().numpy(), _oracle_packed(ws))
    run.close()


def test_peer_merge_cooperative_launch_fallback(monkeypatch):
    """Without a cooperative launch (COMPASS_SCAN_NOCOOP stands in for a refused one) the scan
    runs plain and one k_peer_push follows it: same merged buffer, one more launch per table."""
    import datagen
    import paper_2102_02440_b200 as pb
    from paper_2102_02440_b200.query import QueryRun
    dev = torch.device("cuda", 0)
    ws = datagen.c5(scale=2e-4, w=128, wm=64)
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    counts = {}
    for mode in ("coop", "fallback"):
        if mode == "fallback":
            monkeypatch.setenv("COMPASS_SCAN_NOCOOP", "1")
        run = QueryRun(ws, dev, merge="peer")
        for _ in range(2):   # second pass: lookup tables cached
            run.zero_()
            l0 = pb.kernel_launches()
            for t in ws.tables:
                run.build_table(t.name, data[t.name], datagen.resolve_preds(ws, t.name))
            counts[mode] = pb.kernel_launches() - l0
            run.allreduce()
        torch.cuda.synchronize()
        assert np.array_equal(run.buffer.cpu().numpy(), _oracle_packed(ws))
        run.close()
    assert counts["fallback"] == counts["coop"] + len(ws.tables)


def test_peer_push_histogram_epilogue_not_fused():
    """A hinted key domain sends the 1-D sketches through the histogram epilogue after the
    scan: the push must follow the epilogue (not fused), and the merged counters are exact."""
    import paper_2102_02440_b200 as pb
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11)
    n = 200_000
    z = torch.from_numpy((rng.zipf(1.3, n) % 3000).astype(np.int64)).to(dev)
    p = torch.from_numpy(rng.integers(0, 1000, n).astype(np.int32)).to(dev)
    part = torch.zeros(2 + 5 * 1024, dtype=torch.int64, device=dev)
    sk = pb.Sketch(5, [1024], ["A.z|B.z"], 42, dev, counters=part[2:].view(5, 1024))
    merged = pb.IpcBuffer(part.numel(), dev)
    pb.sketch_update_filtered([z, p], n, [(1, pb.RANGE, 0, 699)], [(sk, [0])], survivors=part[:1],
                              domains=[3000, 0], push=(part[2:], [merged.ptr + 16]))
    torch.cuda.synchronize()
    import oracle
    mask, cnt = oracle.filter_mask({"z": z.cpu().numpy(), "p": p.cpu().numpy()}, [("p", pb.RANGE, 0, 699)])
    ref = oracle.build([z.cpu().numpy()], mask, 5, [1024], ["A.z|B.z"], master=42).reshape(-1)
    got = merged.tensor.cpu().numpy()
    assert np.array_equal(got[2:], ref) and np.array_equal(part[2:].cpu().numpy(), ref)
    assert int(part[0]) == cnt
    sk.close()
    merged.close()


def _worker(rank, world, port, cfg, out_path, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    gpu = rank if torch.cuda.device_count() >= world else 0
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    ws = getattr(datagen, cfg[0])(**cfg[1])
    run = QueryRun(ws, dev, merge="peer", peer_mode=mode)
    assert run.merge.mode == mode
    data = {t.name: datagen.generate_table(ws, t.name, dev, rank=rank, world=world) for t in ws.tables}
    bufs = []
    for _ in range(2):   # two steps: zero + barrier, fused scans + pushes, survivors, barrier
        run.zero_()
        for t in ws.tables:
            run.build_table(t.name, data[t.name], datagen.resolve_preds(ws, t.name))
        run.allreduce()
        torch.cuda.synchronize()
        bufs.append(run.buffer.cpu())
    plan = run.graph().plan_greedy() if ws.kind == "graph" else None
    res = [None] * world
    dist.all_gather_object(res, {"bufs": bufs, "plan": plan})
    if rank == 0:
        torch.save(res, out_path)
    dist.barrier()
    run.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "all"), (2, "owner"), (3, "owner")])
@pytest.mark.parametrize("cfg", [("c5", {"scale": 2e-4, "w": 128, "wm": 64}), ("c4", {"scale": 0.002})])
def test_peer_merge_ranks(cfg, world, mode, tmp_path):
    """Two or three ranks (one GPU each, or processes sharing the pool's one GPU): each builds
    its row shard and pushes into every merged buffer ("all") or into the owners' ranges then
    gathers ("owner", reduce-scatter + all-gather over peer memory); every merged buffer equals
    the oracle's full build, plans agree."""
    import datagen
    out = str(tmp_path / "peer.pt")
    mp.start_processes(_worker, args=(world, _free_port(), cfg, out, mode), nprocs=world, join=True,
                       start_method="spawn")
    res = torch.load(out)
    ref = _oracle_packed(getattr(datagen, cfg[0])(**cfg[1]))
    for r in res:
        for b in r["bufs"]:
            assert np.array_equal(b.numpy(), ref)
    assert all(r["plan"] == res[0]["plan"] for r in res)
