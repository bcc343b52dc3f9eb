"""Row-sharded merge and composition (SURVEY.md §8(e) lever iii, §8(f) 4 second half).

The d rows of a Fast-AGMS sketch are independent until the median (Est =
median_r E_r), so after the scans the partial sketches need not be all-reduced: a
reduce-scatter by sketch row gives rank i the merged rows [r0_i, r1_i) of every sketch, rank i
evaluates E_r of each sub-plan for its rows only, and one all-gather of those per-row exact
integers per greedy level lets every rank take the same medians and make the same choice.
The collective moves half the bytes of the all-reduce and the composition divides by
min(d, N).

Host logic (layout, row ranges, the greedy over gathered rows) is separated from the device
work so it runs under gloo on CPU (tests/test_multirank_gloo.py); on GPUs the per-row values
come from the library's exact estimator on row-shard sketches (caller-owned counter views of
the received chunk).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def row_ranges(d: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges, remainder one row each to the low ranks (ranks >= d get none)."""
    base, rem = divmod(d, world)
    out, r = [], 0
    for i in range(world):
        n = base + (1 if i < rem else 0)
        out.append((r, r + n))
        r += n
    return out


def shard_rows(d: int, world: int) -> int:
    """Rows per rank in the exchanged chunk: max rows of any rank, rounded up to odd (a
    sketch handle needs odd d; the padding rows stay zero and their values are dropped)."""
    R = -(-d // world)
    return R if R % 2 else R + 1


def chunk_layout(cells: list[int], R: int) -> tuple[int, list[int]]:
    """Offsets of each sketch's [R][cells] block inside one rank's chunk; chunk length."""
    offs, o = [], 0
    for c in cells:
        offs.append(o)
        o += R * c
    return o, offs


def pack_rows(counters: list[torch.Tensor], d: int, world: int) -> torch.Tensor:
    """Send buffer of the reduce-scatter: world chunks, chunk i = rows [r0_i, r1_i) of every
    sketch (zero rows up to the odd chunk height R), sketch-major inside the chunk."""
    R = shard_rows(d, world)
    cells = [c[0].numel() for c in counters]
    clen, offs = chunk_layout(cells, R)
    send = torch.zeros(world * clen, dtype=counters[0].dtype, device=counters[0].device)
    for i, (r0, r1) in enumerate(row_ranges(d, world)):
        for c, o, n in zip(counters, offs, cells):
            if r1 > r0:
                send[i * clen + o:i * clen + o + (r1 - r0) * n].copy_(c[r0:r1].reshape(-1))
    return send


def reduce_scatter_rows(counters: list[torch.Tensor], d: int, group=None) -> torch.Tensor:
    """This rank's merged chunk (int64 SUM of every rank's partial rows; exact)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    send = pack_rows(counters, d, world)
    clen = send.numel() // world
    out = torch.empty(clen, dtype=send.dtype, device=send.device)
    if world > 1:
        dist.reduce_scatter_tensor(out, send, op=dist.ReduceOp.SUM, group=group)
    else:
        out.copy_(send)
    return out


def median_card(rows: list[int], n_tables: int, survivors: int) -> float:
    """card(S) of the greedy: survivors for a singleton, else max(Est, 0) with
    Est = median of the d exact row values (element (d-1)/2 of the ascending sort), rounded
    once to fp64."""
    if n_tables == 1:
        return float(survivors)
    v = sorted(rows)[(len(rows) - 1) // 2]
    return max(float(v), 0.0)


def plan_greedy_gathered(tables: dict, edges: list, rows_of_batch, gather):
    """Greedy left-deep plan over row-sharded estimates.

    tables: {alias: survivors}; edges: [(edge_id, u, v)];
    rows_of_batch(list of sub-plans) -> this rank's exact row values per sub-plan (list of
    lists, its own rows only); gather(local) -> the list of every rank's `local`, rank order.
    Each level evaluates its candidates as one batch and gathers once; every rank then holds
    all d rows, takes the same medians and picks the same table.  Same order, prefix cards
    and cost as a single-device plan_greedy on the merged sketches."""
    cache = {}

    def cards(subsets):
        need = [tuple(sorted(S)) for S in subsets if len(S) > 1 and tuple(sorted(S)) not in cache]
        need = list(dict.fromkeys(need))
        local = rows_of_batch(need) if need else []
        parts = gather(local)
        for k, S in enumerate(need):
            rows = [v for p in parts for v in p[k]]
            cache[S] = median_card(rows, len(S), 0)
        out = []
        for S in subsets:
            S = tuple(sorted(S))
            out.append(float(tables[S[0]]) if len(S) == 1 else cache[S])
        return out

    names = sorted(tables)
    if len(names) == 1:
        c = float(tables[names[0]])
        return names, [c], c
    pairs = sorted({tuple(sorted((u, v))) for _, u, v in edges})
    pc = cards(pairs)
    best = min(zip(pc, pairs))[1]
    source = min(best, key=lambda a: (tables[a], a))
    C = [source]
    prefix = [float(tables[source])]
    cost = prefix[0]
    while len(C) < len(names):
        cand = sorted({b for _, u, v in edges for a, b in ((u, v), (v, u)) if a in C and b not in C})
        cc = cards([C + [x] for x in cand])
        c, v = min(zip(cc, cand))
        C.append(v)
        prefix.append(c)
        cost += c
    return C, prefix, cost


def gather_objects(group=None):
    """gather(local) for plan_greedy_gathered over a torch.distributed group (one
    all_gather_object per level; exact Python integers)."""
    def g(local):
        if not (dist.is_initialized() and dist.get_world_size(group) > 1):
            return [local]
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, local, group=group)
        return out
    return g
