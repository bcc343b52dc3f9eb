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

from . import JoinGraph, Sketch, sketch_update_filtered


def packed_layout(q):
    """Layout of the packed int64 buffer of one query: survivors[n_tables] first, then
    every sketch's counters (row-major [d][w0](w1)), each starting 16-byte aligned.
    Returns (total_len, [(offset, count) per sketch])."""
    off = len(q.tables)
    off += off & 1
    out = []
    for s in q.sketches:
        n = s.d
        for w in s.w:
            n *= w
        out.append((off, n))
        off += n + (n & 1)
    return off, out


def allreduce_packed(buffer: torch.Tensor, group=None):
    """Cross-rank merge of partial sketches + survivor counts: one int64 SUM all-reduce
    (exact: integer addition is associative)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buffer, op=dist.ReduceOp.SUM, group=group)
    return buffer


class QueryRun:
    def __init__(self, q, device="cuda", use_domains=True):
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

    def zero_(self):
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
        sketch_update_filtered(cols, n_rows, pr, targets, survivors=self.survivors[ti:ti + 1], stream=stream,
                               domains=domains)

    def build(self, data: dict, preds: dict, stream=None):
        for name in self.tnames:
            self.build_table(name, data[name], preds[name], stream=stream)

    def allreduce(self, group=None):
        """Cross-GPU merge of all partial sketches and survivor counts: one int64 SUM (NCCL)."""
        allreduce_packed(self.buffer, group)

    def sketch_of(self, table: str, edge_ids) -> Sketch:
        for s, sk in zip(self.q.sketches, self.sketches):
            if s.table == table and list(s.edge_ids) == list(edge_ids):
                return sk
        raise KeyError((table, edge_ids))

    def graph(self, survivors=None) -> JoinGraph:
        if survivors is None:
            survivors = self.survivors.tolist()
        # graph vertices in alias order: index order is the tie-break order of plan_greedy
        gnames = sorted(self.tnames)
        surv_by = dict(zip(self.tnames, survivors))
        tix = {n: i for i, n in enumerate(gnames)}
        edges = []
        if getattr(self.q, "kind", "graph") == "selfjoin":
            # self-join size per key sketch (F2): the sketch meets itself on one edge
            names, surv, mats = [], [], []
            for s, sk in zip(self.q.sketches, self.sketches):
                i = len(names)
                names += [f"{s.table}.{s.key_cols[0]}", f"{s.table}.{s.key_cols[0]}'"]
                surv += [surv_by[s.table]] * 2
                edges.append((i, i + 1, sk, sk))
            return JoinGraph(names, surv, edges, mats)
        for eid, u, v in self.q.edges:
            edges.append((tix[u], tix[v], self.sketch_of(u, [eid]), self.sketch_of(v, [eid])))
        mats = []
        for s, sk in zip(self.q.sketches, self.sketches):
            if len(s.edge_ids) == 2:
                eids = [e[0] for e in self.q.edges]
                mats.append((tix[s.table], eids.index(s.edge_ids[0]), eids.index(s.edge_ids[1]), sk))
        return JoinGraph(gnames, [surv_by[n] for n in gnames], edges, mats)

    def close(self):
        for sk in self.sketches:
            sk.close()
