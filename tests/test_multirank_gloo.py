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


# ------------------------------------------------------------------ row-sharded merge + composition (§8(e) iii)
def _worker_rowshard(rank, world, port, cfg, out_path):
    """Partial sketches of this rank's table rows -> reduce-scatter by sketch row -> exact
    per-row values of this rank's rows from its shard only -> greedy over gathered rows."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    import oracle
    from paper_2102_02440_b200 import rowshard as rs
    from paper_2102_02440_b200.query import packed_layout
    ws = getattr(datagen, cfg[0])(**cfg[1])
    buf, names = _build_packed(ws, rank, world)
    _, lay = packed_layout(ws)
    d = ws.sketches[0].d
    views = [buf[o:o + n].view(s.d, *s.w) for (o, n), s in zip(lay, ws.sketches)]
    chunk = rs.reduce_scatter_rows(views, d)
    surv = buf[:len(names)].clone()
    dist.all_reduce(surv, op=dist.ReduceOp.SUM)
    R = rs.shard_rows(d, world)
    cells = [v[0].numel() for v in views]
    _, offs = rs.chunk_layout(cells, R)
    r0, r1 = rs.row_ranges(d, world)[rank]
    vec, mat = {}, {}
    for s, o, n in zip(ws.sketches, offs, cells):
        arr = chunk[o:o + R * n].view(R, *s.w).numpy()
        if len(s.w) == 1:
            vec[(s.table, s.edge_ids[0])] = arr
        else:
            mat[(s.table, tuple(s.edge_ids))] = arr
    tables = dict(zip(names, [int(x) for x in surv.tolist()]))
    shard_graph = oracle.Graph(tables, ws.edges, vec, mat)

    def rows_of_batch(subsets):
        return [oracle.estimate_rows(shard_graph, S)[:r1 - r0] for S in subsets]
    plan = rs.plan_greedy_gathered(tables, ws.edges, rows_of_batch, rs.gather_objects())
    # this rank's rows of every 2- and 3-table connected sub-plan, for the parent's check
    subs = [S for S in oracle.connected_subplans(shard_graph) if 2 <= len(S) <= 3]
    mine = {S: oracle.estimate_rows(shard_graph, S)[:r1 - r0] for S in subs}
    allp = [None] * world
    dist.all_gather_object(allp, (r0, r1, mine))
    if rank == 0:
        torch.save({"plan": plan, "rows": allp}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg", [("c5", {"scale": 5e-5, "w": 64, "wm": 32}),
                                 ("c5", {"scale": 5e-5, "w": 64, "wm": 32, "cycle": True}),
                                 ("c2", {"scale": 2e-4})])
def test_row_sharded_merge_and_greedy_equal_single_device(cfg, world, tmp_path):
    """Reduce-scatter by sketch row + row-sharded composition (SURVEY.md §8(e) lever iii):
    every rank's rows of every sub-plan equal the single-device oracle's rows, and the
    greedy plan from gathered rows equals oracle.plan_greedy on the merged sketches."""
    import datagen
    import oracle
    from paper_2102_02440_b200.query import packed_layout
    out = str(tmp_path / "rs.pt")
    mp.start_processes(_worker_rowshard, args=(world, _free_port(), cfg, out), nprocs=world, join=True,
                       start_method="spawn")
    res = torch.load(out)
    ws = getattr(datagen, cfg[0])(**cfg[1])
    single, names = _build_packed(ws, 0, 1)
    _, lay = packed_layout(ws)
    vec, mat = {}, {}
    for (o, n), s in zip(lay, ws.sketches):
        arr = single[o:o + n].view(s.d, *s.w).numpy()
        if len(s.w) == 1:
            vec[(s.table, s.edge_ids[0])] = arr
        else:
            mat[(s.table, tuple(s.edge_ids))] = arr
    og = oracle.Graph(dict(zip(names, [int(x) for x in single[:len(names)].tolist()])), ws.edges, vec, mat)
    for r0, r1, mine in res["rows"]:
        for S, rows in mine.items():
            assert rows == oracle.estimate_rows(og, S)[r0:r1], (S, r0, r1)
    assert tuple(res["plan"][0]) == tuple(oracle.plan_greedy(og)[0])
    assert res["plan"][1] == oracle.plan_greedy(og)[1]


def test_row_ranges_and_pack_layout():
    from paper_2102_02440_b200 import rowshard as rs
    for d in (1, 5, 7, 9):
        for world in (1, 2, 3, 8):
            rr = rs.row_ranges(d, world)
            assert rr[0][0] == 0 and rr[-1][1] == d and all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
            assert max(b - a for a, b in rr) - min(b - a for a, b in rr) <= 1
            R = rs.shard_rows(d, world)
            assert R % 2 == 1 and R >= max(b - a for a, b in rr)
    c = [torch.arange(5 * 4).view(5, 4), 100 + torch.arange(5 * 6).view(5, 2, 3)]
    send = rs.pack_rows(c, 5, 2)   # ranks get rows [0,3) and [3,5); R = 3
    clen = send.numel() // 2
    assert clen == 3 * 4 + 3 * 6
    assert torch.equal(send[:12], c[0][0:3].reshape(-1)) and torch.equal(send[12:30], c[1][0:3].reshape(-1))
    assert torch.equal(send[30:38], c[0][3:5].reshape(-1)) and torch.equal(send[38:42], torch.zeros(4, dtype=send.dtype))
    assert torch.equal(send[42:54], c[1][3:5].reshape(-1)) and torch.equal(send[54:60], torch.zeros(6, dtype=send.dtype))


# ---- merge over peer memory (query.PeerMerge, SURVEY.md §8(f) 4 P2P variant): host logic with
# the library's IPC buffers and push emulated by file-backed shared tensors.  A "device
# pointer" is (rank + 1) << 40 plus a byte offset, so the slice arithmetic of PeerMerge
# (ptr + 8 * offset) is exercised as on the device.
class _FakeIpc:
    def __init__(self, numel, device, root, rank):
        self.numel = numel
        path = os.path.join(root, f"merged{rank}.bin")
        self.tensor = torch.from_file(path, shared=True, size=numel, dtype=torch.int64)
        self.tensor.zero_()
        self.ptr = (rank + 1) << 40
        self.handle = path.encode()
        _LOCKS[self.ptr] = path + ".lock"

    def close(self):
        pass


def _fake_open(handle, device, numel):
    path = handle.decode()
    rank = int(os.path.basename(path)[len("merged"):-len(".bin")])
    _FAKE[(rank + 1) << 40] = torch.from_file(path, shared=True, size=numel, dtype=torch.int64)
    _LOCKS[(rank + 1) << 40] = path + ".lock"
    return (rank + 1) << 40


_FAKE = {}


def _owner_lo(total, peers, o):
    return total if o >= peers else (total * o // peers) & ~1


def _fake_push(src, dst_ptrs, stream=None, owner=None):
    """red.add emulation: the read-modify-write of another process's buffer under a file lock
    (the device's atomics need none).  owner = (rank, offset, total): each element only to the
    rank owning its range (the library's owner mode, csrc/peer.cuh)."""
    import fcntl
    n = src.numel()
    for q, p in enumerate(dst_ptrs):
        base = (p >> 40) << 40
        off = (p - base) // 8
        a, b = 0, n
        if owner is not None:   # this rank's share of src owned by rank q
            _, o0, total = owner
            a = max(0, _owner_lo(total, len(dst_ptrs), q) - o0)
            b = min(n, _owner_lo(total, len(dst_ptrs), q + 1) - o0)
            if a >= b:
                continue
        with open(_LOCKS[base], "a") as lk:
            fcntl.flock(lk, fcntl.LOCK_EX)
            _FAKE[base][off + a:off + b] += src[a:b]
            fcntl.flock(lk, fcntl.LOCK_UN)


def _fake_gather(dst_ptrs, rank, total, stream=None):
    own = _FAKE[dst_ptrs[rank]]
    for q, p in enumerate(dst_ptrs):
        if q != rank:
            a, b = _owner_lo(total, len(dst_ptrs), q), _owner_lo(total, len(dst_ptrs), q + 1)
            own[a:b] = _FAKE[p][a:b]


_LOCKS = {}


def _worker_peer(rank, world, port, cfg, root, out_path, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    from paper_2102_02440_b200 import query
    from paper_2102_02440_b200.query import PeerMerge, table_slices
    ws = getattr(datagen, cfg[0])(**cfg[1])
    part, _ = _build_packed(ws, rank, world)
    numel = part.numel()

    def fake_ipc(n, device):
        b = _FakeIpc(n, device, root, rank)
        _FAKE[b.ptr] = b.tensor
        return b

    query.IpcBuffer = fake_ipc
    query.ipc_open = lambda h, device: _fake_open(h, device, numel)
    query.ipc_close = lambda p: None
    query.sketch_peer_push = _fake_push
    query.sketch_peer_gather = _fake_gather
    buf = torch.zeros_like(part)
    m = PeerMerge(buf, len(ws.tables), table_slices(ws), mode=mode)
    outs = []
    for _ in range(2):   # two steps: zero + barrier, per-table pushes (as the fused scan does), finish
        m.zero_()
        buf.copy_(part)
        for t in ws.tables:
            if t.name in m.slices:
                _fake_push(*m.push_for(t.name))
        m.finish()
        outs.append(buf.clone())
    if rank == 0:
        torch.save(outs, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["all", "owner"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg", [("c1", {"scale": 0.2}), ("c5", {"scale": 5e-5, "w": 64, "wm": 32})])
def test_peer_merge_host_logic_equals_single_build(cfg, world, mode, tmp_path):
    """Every rank's merged buffer after the pushes == the single-process build, two steps in a
    row (the merged buffers are re-zeroed behind a barrier)."""
    import datagen
    out = str(tmp_path / "peer.pt")
    mp.start_processes(_worker_peer, args=(world, _free_port(), cfg, str(tmp_path), out, mode), nprocs=world,
                       join=True, start_method="spawn")
    outs = torch.load(out)
    ws = getattr(datagen, cfg[0])(**cfg[1])
    full, _ = _build_packed(ws, 0, 1)
    for b in outs:
        assert torch.equal(b, full)
