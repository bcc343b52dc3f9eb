"""Query-level driver of the hot path: one fused scan per table, one packed int64
buffer for all sketches and survivor counts (so the cross-GPU merge is a single
NCCL all-reduce, PAPER.md:86 / SURVEY.md §8(e)), then composition + greedy plan.

The query description is duck-typed (``datagen.Workload`` satisfies it):
  q.tables   : objects with .name, .cols (objects with .name, .dtype), .preds
  q.edges    : (edge_id, table_u, table_v)
  q.sketches : objects with .table, .key_cols, .edge_ids, .d, .w
  q.master_seed
Predicates passed to ``build`` are already resolved: (col_name, kind, lo, hi, set).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (IpcBuffer, JoinGraph, Sketch, ipc_close, ipc_open, sketch_peer_gather, sketch_peer_push,
               sketch_update_filtered, sketch_wire_pack, sketch_wire_unpack)


def packed_layout(q):
    """Layout of the packed int64 buffer of one query: survivors[n_tables] first, then every
    sketch's counters (row-major [d][w0](w1)) grouped by table in table order, each starting
    16-byte aligned, so one table's sketches form one contiguous slice (per-table all-reduce).
    Returns (total_len, [(offset, count) per sketch, in q.sketches order])."""
    off = len(q.tables)
    off += off & 1
    out = [None] * len(q.sketches)
    for t in q.tables:
        for i, s in enumerate(q.sketches):
            if s.table != t.name:
                continue
            n = s.d
            for w in s.w:
                n *= w
            out[i] = (off, n)
            off += n + (n & 1)
    return off, out


def table_slices(q):
    """{table: (start, end)} of each table's sketches in the packed buffer."""
    _, lay = packed_layout(q)
    sl = {}
    for (o, n), s in zip(lay, q.sketches):
        a, b = sl.get(s.table, (o, o + n))
        sl[s.table] = (min(a, o), max(b, o + n + (n & 1)))
    return sl


def allreduce_packed(buffer: torch.Tensor, group=None):
    """Cross-rank merge of partial sketches + survivor counts: one int64 SUM all-reduce
    (exact: integer addition is associative)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buffer, op=dist.ReduceOp.SUM, group=group)
    return buffer


class PackedMerge:
    """Cross-GPU merge of one query's packed buffer, when a
    process group of > 1 rank is initialised:
      wire="i64": the slices are summed with NCCL as int64;
      wire="i32": each slice is packed to int32 (pack(src64, dst32): the library's
                  sketch_wire_pack), summed, and unpacked (exact while every table has < 2^31
                  rows, which the caller checks; lever i);
      overlap=True: each table's slice is all-reduced asynchronously as soon as its scan is
                  enqueued (reduce_table), on NCCL's stream, while the next table scans (lever
                  ii); finish() then only merges the survivor counts and waits.
    Host logic only (the packing kernels are passed in), so it runs under gloo on CPU too."""

    def __init__(self, buffer, n_tables, slices, wire="i64", overlap=False, group=None, pack=None, unpack=None,
                 always=False):
        assert wire in ("i64", "i32")
        self.buffer, self.slices, self.wire, self.overlap, self.group = buffer, slices, wire, overlap, group
        self.always = always   # run the collectives even for a group of one rank (tests)
        self.n_s = n_tables + (n_tables & 1)
        self.pack, self.unpack = pack, unpack
        self.wire_buf = torch.empty(buffer.numel(), dtype=torch.int32, device=buffer.device) if wire == "i32" else None
        self.pending = []

    def world(self) -> int:
        if dist.is_available() and dist.is_initialized():
            n = dist.get_world_size(self.group)
            return 2 if (self.always and n == 1) else n
        return 1

    def _reduce(self, a: int, b: int, async_op: bool):
        if self.wire == "i32":
            w = self.wire_buf[a:b]
            self.pack(self.buffer[a:b], w)
            return (dist.all_reduce(w, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op), a, b)
        return (dist.all_reduce(self.buffer[a:b], op=dist.ReduceOp.SUM, group=self.group, async_op=async_op), None, None)

    def _wait(self, item):
        work, a, b = item
        if work is not None:
            work.wait()
        if a is not None:
            self.unpack(self.wire_buf[a:b], self.buffer[a:b])

    def reduce_table(self, name: str):
        """Called right after table `name`'s scan was enqueued."""
        if self.overlap and name in self.slices and self.world() > 1:
            a, b = self.slices[name]
            self.pending.append(self._reduce(a, b, async_op=True))

    def finish(self):
        """Every partial merged: the pending per-table reductions (overlap) or the whole sketch
        region, then the survivor counts (int64)."""
        if self.world() <= 1:
            self.pending = []
            return
        if self.overlap:
            for item in self.pending:
                self._wait(item)
            self.pending = []
        else:
            self._wait(self._reduce(self.n_s, self.buffer.numel(), async_op=False))
        dist.all_reduce(self.buffer[:self.n_s], op=dist.ReduceOp.SUM, group=self.group)


class PeerMerge:
    """Cross-GPU merge over peer memory (SURVEY.md §8(f) 4, P2P variant of the fused flush +
    all-reduce).  Every rank owns a merged buffer with the packed layout, allocated
    by the library for CUDA IPC and mapped into every other rank's process (handles exchanged
    with all_gather_object).  Each table's scan is launched with a push of its partial slice
    into that slice of every rank's merged buffer — fused into the scan's cooperative launch
    (after a grid barrier behind the last CTA's flush) where the library can — and finish()
    pushes the survivor counts, waits for the stream, and after a barrier (every rank's pushes
    complete) copies the merged buffer into the partial buffer, so the sketch handles read the
    sums.  No NCCL kernel; exact integer addition in any order.

    mode "all": every element is added into every rank's buffer (one shot, N x the bytes);
    mode "owner" (default from 3 ranks): reduce-scatter — each element goes to the rank owning
    its range of the buffer only — then, after a barrier, every rank reads the other owners'
    ranges (sketch_peer_gather) and a second barrier keeps the owners' buffers untouched until
    every rank has read them: 2 (N-1)/N x the bytes, like a ring all-reduce."""

    def __init__(self, buffer, n_tables, slices, group=None, mode=None):
        self.buffer, self.slices, self.group = buffer, slices, group
        self.n_s = n_tables + (n_tables & 1)
        self.init = dist.is_available() and dist.is_initialized()
        self.world_n = dist.get_world_size(group) if self.init else 1
        rank = dist.get_rank(group) if self.init else 0
        assert self.world_n <= 8, "peer merge: at most 8 ranks"
        self.rank = rank
        self.mode = mode or ("owner" if self.world_n >= 3 else "all")
        assert self.mode in ("all", "owner")
        self.final = IpcBuffer(buffer.numel(), buffer.device)
        handles = [None] * self.world_n
        if self.world_n > 1:
            dist.all_gather_object(handles, self.final.handle, group=group)
        self.opened = []
        self.ptrs = []
        for r in range(self.world_n):
            if r == rank:
                self.ptrs.append(self.final.ptr)
            else:
                p_ = ipc_open(handles[r], buffer.device)
                self.opened.append(p_)
                self.ptrs.append(p_)
        self.stream = None

    def world(self) -> int:
        return self.world_n

    def _barrier(self, stream):
        if self.world_n > 1:
            if self.buffer.is_cuda:
                (stream or torch.cuda.current_stream(self.buffer.device)).synchronize()
            dist.barrier(group=self.group)

    def zero_(self, stream=None):
        """Zero the partial and this rank's merged buffer; no rank pushes before every rank
        has zeroed (barrier)."""
        self.buffer.zero_()
        self.final.tensor.zero_()
        self._barrier(stream)

    def _owner(self, a):
        return (self.rank, a, self.buffer.numel()) if self.mode == "owner" else None

    def push_for(self, name: str, stream=None):
        self.stream = stream
        a, b = self.slices[name]
        src, dst = self.buffer[a:b], [p + 8 * a for p in self.ptrs]
        own = self._owner(a)
        return (src, dst) if own is None else (src, dst, own)

    def reduce_table(self, name: str):
        pass   # the push travels with the scan

    def finish(self):
        s = self.stream
        sketch_peer_push(self.buffer[:self.n_s], list(self.ptrs), stream=s, owner=self._owner(0))
        self._barrier(s)
        if self.mode == "owner":
            sketch_peer_gather(list(self.ptrs), self.rank, self.buffer.numel(), stream=s)
            self._barrier(s)   # every rank has read the owners' ranges before any rank zeroes
        if not self.buffer.is_cuda:   # (host logic tests with emulated peer buffers)
            self.buffer.copy_(self.final.tensor)
            return
        with torch.cuda.stream(s or torch.cuda.current_stream(self.buffer.device)):
            self.buffer.copy_(self.final.tensor)

    def close(self):
        for p_ in self.opened:
            ipc_close(p_)
        self.opened = []
        self.final.close()


class QueryRun:
    """One query's sketches in one packed int64 buffer; cross-GPU merge by PackedMerge."""

    def __init__(self, q, device="cuda", use_domains=True, wire="i64", overlap=False, group=None, always_merge=False,
                 merge="nccl", peer_mode=None):
        self.q = q
        self.use_domains = use_domains
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.tnames = [t.name for t in q.tables]
        total, lay = packed_layout(q)
        offs = [o for o, _ in lay]
        sizes = [n for _, n in lay]
        self.buffer = torch.zeros(total, dtype=torch.int64, device=self.device)
        self.survivors = self.buffer[:len(self.tnames)]
        self.sketches = []
        for s, o, n in zip(q.sketches, offs, sizes):
            view = self.buffer[o:o + n].view(s.d, *s.w)
            self.sketches.append(Sketch(s.d, s.w, s.edge_ids, q.master_seed, self.device, counters=view))
        self.sketch_bytes = sum(sizes) * 8
        if wire == "i32" and any(t.n_rows >= (1 << 31) for t in q.tables):
            wire = "i64"   # int32 partial/merged counters need < 2^31 rows per table
        assert merge in ("nccl", "peer")
        self.peer = merge == "peer"
        if self.peer:
            self.merge = PeerMerge(self.buffer, len(self.tnames), table_slices(q), group, mode=peer_mode)
        else:
            self.merge = PackedMerge(self.buffer, len(self.tnames), table_slices(q), wire, overlap, group,
                                     pack=lambda a, b: sketch_wire_pack(a, b),
                                     unpack=lambda a, b: sketch_wire_unpack(a, b), always=always_merge)

    def zero_(self, stream=None):
        if self.peer:
            self.merge.zero_(stream)
        else:
            self.buffer.zero_()

    def build_table(self, name: str, columns: dict, preds, stream=None):
        """Fused filter + sketch update for every sketch of table `name` (one scan)."""
        t = next(t for t in self.q.tables if t.name == name)
        cnames = [c.name for c in t.cols]
        cols = [columns[c] for c in cnames]
        n_rows = int(cols[0].shape[0]) if cols else 0
        pr = [(cnames.index(p[0]), p[1], p[2], p[3], p[4] if len(p) > 4 else None) for p in preds]
        targets = [(sk, [cnames.index(k) for k in s.key_cols])
                   for s, sk in zip(self.q.sketches, self.sketches) if s.table == name]
        ti = self.tnames.index(name)
        domains = [getattr(c, "domain", 0) or 0 for c in t.cols] if self.use_domains else None
        push = self.merge.push_for(name, stream) if (self.peer and name in self.merge.slices) else None
        sketch_update_filtered(cols, n_rows, pr, targets, survivors=self.survivors[ti:ti + 1], stream=stream,
                               domains=domains, push=push)
        self.merge.reduce_table(name)

    def build(self, data: dict, preds: dict, stream=None):
        for name in self.tnames:
            self.build_table(name, data[name], preds[name], stream=stream)

    def allreduce(self):
        """Cross-GPU merge of all partial sketches and survivor counts (NCCL SUM)."""
        self.merge.finish()

    def sketch_of(self, table: str, edge_ids) -> Sketch:
        for s, sk in zip(self.q.sketches, self.sketches):
            if s.table == table and list(s.edge_ids) == list(edge_ids):
                return sk
        raise KeyError((table, edge_ids))

    def graph(self, survivors=None, sketches=None) -> JoinGraph:
        """JoinGraph over the merged sketches (or `sketches`, one per q.sketches entry, e.g.
        the row shards of merge_rows)."""
        if survivors is None:
            survivors = self.survivors.tolist()
        if sketches is None:
            sketches = self.sketches
        # graph vertices in alias order: index order is the tie-break order of plan_greedy
        gnames = sorted(self.tnames)
        surv_by = dict(zip(self.tnames, survivors))
        tix = {n: i for i, n in enumerate(gnames)}
        edges = []
        if getattr(self.q, "kind", "graph") == "selfjoin":
            # self-join size per key sketch (F2): the sketch meets itself on one edge
            names, surv, mats = [], [], []
            for s, sk in zip(self.q.sketches, sketches):
                i = len(names)
                names += [f"{s.table}.{s.key_cols[0]}", f"{s.table}.{s.key_cols[0]}'"]
                surv += [surv_by[s.table]] * 2
                edges.append((i, i + 1, sk, sk))
            return JoinGraph(names, surv, edges, mats)
        def sk_of(table, eids):
            for s, sk in zip(self.q.sketches, sketches):
                if s.table == table and list(s.edge_ids) == list(eids):
                    return sk
            raise KeyError((table, eids))
        for eid, u, v in self.q.edges:
            edges.append((tix[u], tix[v], sk_of(u, [eid]), sk_of(v, [eid])))
        mats = []
        for s, sk in zip(self.q.sketches, sketches):
            if len(s.edge_ids) >= 2:   # matrices and 3-D tensors
                eids = [e[0] for e in self.q.edges]
                mats.append((tix[s.table], eids.index(s.edge_ids[0]), eids.index(s.edge_ids[1]), sk))
        return JoinGraph(gnames, [surv_by[n] for n in gnames], edges, mats)

    # ---- row-sharded merge and composition (SURVEY.md §8(e) lever iii; rowshard.py)
    def merge_rows(self, group=None):
        """Reduce-scatter by sketch row instead of the all-reduce: this rank receives the
        merged rows row_ranges(d, N)[rank] of every sketch (plus zero rows up to an odd count)
        and the merged survivor counts.  Returns (row-shard Sketch per q.sketches entry,
        own row count)."""
        import torch.distributed as dist
        from . import rowshard as rs
        d = self.q.sketches[0].d
        assert all(s.d == d for s in self.q.sketches), "row sharding needs one d for the query"
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        chunk = rs.reduce_scatter_rows([sk.counters for sk in self.sketches], d, group)
        if world > 1:
            dist.all_reduce(self.survivors, op=dist.ReduceOp.SUM, group=group)
        R = rs.shard_rows(d, world)
        cells = [sk.counters[0].numel() for sk in self.sketches]
        _, offs = rs.chunk_layout(cells, R)
        shards = []
        for s, o, n in zip(self.q.sketches, offs, cells):
            shards.append(Sketch(R, s.w, s.edge_ids, self.q.master_seed, self.device,
                                 counters=chunk[o:o + R * n].view(R, *s.w)))
        self._row_chunk = chunk   # keeps the views alive
        r0, r1 = rs.row_ranges(d, world)[rank]
        return shards, r1 - r0

    def plan_greedy_rowshard(self, shards, own_rows: int, group=None):
        """Greedy plan from row-sharded estimates: each level's candidate sub-plans are
        evaluated on this rank's rows (exact per-row values), one all-gather per level."""
        from . import rowshard as rs
        surv = dict(zip(self.tnames, self.survivors.tolist()))
        g = self.graph(survivors=[surv[n] for n in self.tnames], sketches=shards)

        def rows_of_batch(subsets):
            if own_rows == 0:
                return [[] for _ in subsets]
            return [g.estimate_join_exact(S)[:own_rows] for S in subsets]
        return rs.plan_greedy_gathered(surv, self.q.edges, rows_of_batch, rs.gather_objects(group))

    def close(self):
        for sk in self.sketches:
            sk.close()
        if self.peer:
            self.merge.close()
