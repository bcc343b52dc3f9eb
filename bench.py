#!/usr/bin/env python
"""Benchmark of the COMPASS hot path on B200 (BASELINE.json metric:
"filtered sketch-build tuples/s and % of HBM GB/s at 1/2/4/8 B200").

A *step* is one pass of the whole hot path over the workload's tables, inputs
resident in HBM: zero the packed sketch buffer, one fused filter+hash+update
scan per table (sketch_update_filtered), the cross-GPU merge (N>1: per-table int32
all-reduces overlapped with the next scan), the composition estimates of the
connected sub-plans the planner reads (estimate_join) and the greedy plan
(plan_greedy).  value = rows scanned by all ranks / t_build, t_build = first kernel
of the step -> final int64 sketches resident after the merge, max
over ranks, CUDA events; the full step time is ms_per_step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl reference]

Default workload: C4 (BASELINE.json configs[3]: 1e9-row fact table, int64 Zipf-1.5
keys, 3 conjunctive ranges, d=9 x w=16384 sketches on 2 join attributes), the
metric's 1/2/4/8-GPU configuration that fits one B200.
Inputs (28 GB) exceed L2 (126 MB) between steps; no flush is needed.
The oracle (oracle/) is executed only in the cpu_baseline leg and --impl reference.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "filtered sketch-build tuples/s and % of HBM GB/s at 1/2/4/8 B200"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def _workload(name: str, scale: float):
    if name == "C5":
        return datagen.c5(scale=scale)
    if name == "C5-cycle":
        return datagen.c5(scale=scale, cycle=True)
    return datagen.CONFIGS[name](scale=scale)


def _subplans(ws):
    """All connected sub-plans with >= 2 tables (plain graph enumeration)."""
    from itertools import combinations
    names = sorted(t.name for t in ws.tables)
    adj = {n: set() for n in names}
    for _, u, v in ws.edges:
        adj[u].add(v)
        adj[v].add(u)
    out = []
    for k in range(2, len(names) + 1):
        for c in combinations(names, k):
            s = set(c)
            seen, st = {c[0]}, [c[0]]
            while st:
                x = st.pop()
                for y in adj[x]:
                    if y in s and y not in seen:
                        seen.add(y)
                        st.append(y)
            if seen == s:
                out.append(c)
    return out


def _torch_mask(cols: dict, preds) -> torch.Tensor:
    """Survivor mask with plain torch ops (used only to count algorithmic bytes, outside timing)."""
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
    return m


def _sectors_hit(mask: torch.Tensor, elem_bytes: int) -> int:
    per = 32 // elem_bytes
    n = mask.shape[0]
    pad = (-n) % per
    mm = torch.cat([mask, torch.zeros(pad, dtype=torch.bool, device=mask.device)]) if pad else mask
    return int(mm.view(-1, per).any(dim=1).sum().item())


def algorithmic_bytes(ws, data, preds, run) -> dict:
    """SURVEY.md §8(d) B_alg: predicate columns in full + key-column 32-B sectors holding
    >= 1 survivor + the final int64 sketch bytes; each column counted once per scan."""
    total, full, per = 0, 0, {}
    for t in ws.tables:
        cols = data[t.name]
        pcols = {p[0] for p in preds[t.name]}
        kcols = {k for s in ws.sketches_of(t.name) for k in s.key_cols} - pcols
        mask = _torch_mask(cols, preds[t.name]) if preds[t.name] else None
        tb = 0
        for c in pcols:
            tb += cols[c].numel() * cols[c].element_size()
        for c in kcols:
            eb = cols[c].element_size()
            tb += cols[c].numel() * eb if mask is None else 32 * _sectors_hit(mask, eb)
        for c in pcols | kcols:
            full += cols[c].numel() * cols[c].element_size()
        for s in ws.sketches_of(t.name):
            cells = 1
            for w in s.w:
                cells *= w
            tb += 8 * s.d * cells
        per[t.name] = tb
        total += tb
    full += run.sketch_bytes
    return {"alg": total, "full": full, "per_table": per}


def binding_roof(ws, survivors, per_table_bytes, kernel_ms, hbm_gbs, roofs) -> dict | None:
    """Per-table binding roof of the scans: sum over tables of max(HBM time of the table's
    algorithmic bytes, its naive counter-update time, its naive hash time) with the measured
    roofs (MEASURED_ROOFS.json).  The lookup-table path (int32 keys with domain hints
    <= 2^22) does no hashing, so its tables take no hash term.  A table whose scan is
    update-bound (C5 T9, cycle T10: every survivor costs d shared atomics per 1-D sketch and
    d L2 red per matrix) cannot reach the HBM roof; this is the roof it can reach."""
    if not roofs:
        return None
    tot, per = 0.0, {}
    for tb, sv in zip(ws.tables, survivors):
        keys = {k for s in ws.sketches_of(tb.name) for k in s.key_cols}
        cmap = {c.name: c for c in tb.cols}
        lut = len(keys) <= 2 and all(cmap[k].dtype == "int32" and 0 < (getattr(cmap[k], "domain", 0) or 0) <= (1 << 22)
                                     for k in keys)
        wide = any(cmap[k].dtype == "int64" for k in keys)
        t_upd = t_hash = 0.0
        for s in ws.sketches_of(tb.name):
            cells = 1
            for w in s.w:
                cells *= w
            u = sv * s.d
            t_upd += u / (roofs["atoms_smem_per_s"] if s.d * cells * 4 <= 96 * 1024 else roofs["red_l2_u64_mat10mb_per_s"])
            if not lut:
                t_hash += u * len(s.w) / (roofs["hash_wide_pairs_per_s"] if wide else roofs["hash_narrow_pairs_per_s"])
        t_hbm = per_table_bytes[tb.name] / (hbm_gbs * 1e9)
        terms = {"hbm": t_hbm, "update": t_upd, "hash": t_hash}
        b = max(terms, key=terms.get)
        per[tb.name] = {"bound": b, "roof_ms": round(terms[b] * 1e3, 4)}
        tot += terms[b]
    return {"roof_time_ms": round(tot * 1e3, 4), "frac": round(tot * 1e3 / kernel_ms, 4), "per_table": per,
            "how": "sum over tables of max(t_hbm, t_update, t_hash) (naive counts, measured roofs)"}


class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except Exception:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _measured_roofs() -> dict:
    """Roofs 2 and 3 of SURVEY.md §8(d) and the read-only stream, measured on a B200 by
    tools/roofs_micro.cu (MEASURED_ROOFS.json, beside the driver's MEASURED_PEAKS.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_ROOFS.json")))
    except Exception:
        return {}


def _int_update_roofs(ws, survivors, kernel_ms, roofs) -> dict:
    """Algorithmic hash and update work of the scans (SURVEY.md §8(d) roofs 2 and 3), counted
    without the exact levers (every survivor hashed and counted once per sketch row):
      hash pairs  I = sum_t survivors_t * sum_{s of t} d_s * ndim_s   ((xi, h) per key and row)
      updates     U = sum_t survivors_t * sum_{s of t} d_s            (counter increments)
    achieved = I / t (U / t) over the scans' time; peak = the measured roof (narrow / wide hash
    path by key width; shared-memory atomics for sketches that fit a CTA, L2 red otherwise).
    frac > 1 means the levers (key aggregation, heavy hitters, histograms, lookup tables)
    beat the naive roof."""
    if not roofs:
        return {"int_frac": None, "update_frac": None, "roofs_source": "MEASURED_ROOFS.json missing"}
    t = kernel_ms / 1e3
    pairs_n = pairs_w = 0
    t_upd = 0.0
    upd = 0
    for tb, sv in zip(ws.tables, survivors):
        wide = any(c.dtype == "int64" for c in tb.cols)
        for s in ws.sketches_of(tb.name):
            cells = 1
            for w in s.w:
                cells *= w
            pr = sv * s.d * len(s.w)
            if wide:
                pairs_w += pr
            else:
                pairs_n += pr
            u = sv * s.d
            upd += u
            fits = s.d * cells * 4 <= 96 * 1024
            t_upd += u / (roofs["atoms_smem_per_s"] if fits else roofs["red_l2_u64_mat10mb_per_s"])
    t_hash = pairs_n / roofs["hash_narrow_pairs_per_s"] + pairs_w / roofs["hash_wide_pairs_per_s"]
    return {"int": {"hash_pairs": pairs_n + pairs_w, "achieved_pairs_per_s": (pairs_n + pairs_w) / t,
                    "roof_time_ms": round(t_hash * 1e3, 4), "frac": round(t_hash / t, 4)},
            "update": {"counter_increments": upd, "achieved_per_s": upd / t,
                       "roof_time_ms": round(t_upd * 1e3, 4), "frac": round(t_upd / t, 4)},
            "int_frac": round(t_hash / t, 4), "update_frac": round(t_upd / t, 4),
            "roofs_source": "MEASURED_ROOFS.json (tools/roofs_micro.cu)"}


def _relaunch(n: int) -> int:
    """`bench.py --gpus N` run as one process: re-executes itself under torchrun with N ranks
    on this node (one process per GPU, NCCL over NVLink), rendezvous on 127.0.0.1."""
    import socket
    if torch.cuda.device_count() < n and not os.environ.get("COMPASS_BENCH_SHARED_GPU"):
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {torch.cuda.device_count()}", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


NCCL_LOG = "/tmp/compass_bench_nccl.%h.%p.log"


def _setup_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and os.environ.get("COMPASS_BENCH_SHARED_GPU"):
        # functional test of the multi-rank bench logic on a one-GPU box (tests/test_bench_ranks_gpu.py):
        # every rank on cuda:0, gloo collectives; the numbers of such a run are not measurements
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        return world, rank, 0
    if world > 1:
        # NCCL's communicator line (rank count, NVLS / channels) is kept so the JSON line can
        # show the collective really spanned every rank
        if "NCCL_DEBUG" not in os.environ:
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
            os.environ["NCCL_DEBUG_FILE"] = NCCL_LOG
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _nccl_comm_line() -> str | None:
    """The 'comm ... nRanks N' INIT line NCCL wrote for this process (NCCL_DEBUG_FILE)."""
    import glob
    import socket
    path = NCCL_LOG.replace("%h", socket.gethostname()).replace("%p", str(os.getpid()))
    for f in [path] + glob.glob("/tmp/compass_bench_nccl.*.%d.log" % os.getpid()):
        try:
            for line in open(f):
                if "nRanks" in line or "nranks" in line:
                    return line.strip()[:300]
        except OSError:
            continue
    return None


def _barrier(world):
    if world > 1:
        dist.barrier()


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _oracle_pass(ws, cols_by_table, preds_by_table, threads: int, out: dict | None = None) -> float:
    """One timed oracle pass (O1 filter + O2/O3 builds, SURVEY.md §8(d) "Oracle timing
    beside it") over the sampled rows.  threads > 1: the rows of every table are split into
    `threads` contiguous ranges, each thread filters and builds private sketches for its range
    (the oracle's C routines run outside the GIL), and the private sketches are merged by int64
    addition (O4).  The oracle's arithmetic is used as it stands."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    def part(tname, a, b):
        cols = {c: v[a:b] for c, v in cols_by_table[tname].items()}
        mask, _ = oracle.filter_mask(cols, preds_by_table[tname])
        return [oracle.build([cols[k] for k in s.key_cols], mask, s.d, s.w, s.edge_ids, master=ws.master_seed)
                for s in ws.sketches_of(tname)]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for t in ws.tables:
            n = len(next(iter(cols_by_table[t.name].values())))
            cuts = [n * i // threads for i in range(threads + 1)]
            parts = list(ex.map(lambda ab: part(t.name, *ab), zip(cuts[:-1], cuts[1:])))
            merged = parts[0]
            for p_ in parts[1:]:
                for m, q in zip(merged, p_):
                    m += q
            if out is not None:
                out[t.name] = merged
    return time.perf_counter() - t0


def cpu_oracle_sample(ws, rows_budget: int, device, threads: int | None = None, single: bool = True) -> dict:
    """Time the oracle (O1 filter + O2/O3 builds) on the first rows of every table
    (proportional sample) on this host: all hardware threads (private sketches merged by
    int64 addition) and, on a smaller sample, single-threaded."""
    cores = threads or os.cpu_count() or 1
    total = ws.total_rows
    frac = min(1.0, rows_budget / total)
    cols, preds, scanned = {}, {}, 0
    for t in ws.tables:
        n = max(1, int(t.n_rows * frac))
        cols[t.name] = {c.name: datagen._gen_column(ws, t, c, 0, n, device).cpu().numpy() for c in t.cols}
        preds[t.name] = datagen.resolve_preds(ws, t.name)
        scanned += n
    t_mt = _oracle_pass(ws, cols, preds, cores)
    out = {"value": scanned / t_mt, "unit": "tuples/s", "cores": cores, "kind": "oracle", "seconds": round(t_mt, 4),
           "sample": f"first {frac:.3%} of every table of {ws.name} ({scanned} rows), filter + sketch builds, "
                     f"plain C oracle on {cores} threads (row ranges, private sketches merged by int64 addition), "
                     f"{t_mt:.1f} s"}
    if single:
        # single-threaded leg on the first 1/cores of the same sample (bounded CPU time)
        frac1 = 1.0 / cores
        cols1 = {tn: {c: v[:max(1, int(len(v) * frac1))] for c, v in cc.items()} for tn, cc in cols.items()}
        scanned1 = sum(len(next(iter(cc.values()))) for cc in cols1.values())
        t_st = _oracle_pass(ws, cols1, preds, 1)
        out["single_thread"] = {"value": scanned1 / t_st, "unit": "tuples/s", "cores": 1,
                                "sample": f"first {scanned1} rows of the same sample, {t_st:.1f} s"}
    return out


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, on this host's cores."""
    if rank != 0:
        return
    ws = _workload(args.workload, args.scale)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    budget = args.ref_rows
    samples, secs = [], []
    base = None
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(ws, budget, dev, single=False)
        if i >= args.warmup:
            samples.append(r["value"])
            secs.append(r["seconds"])
        base = r
    v = sorted(samples)[len(samples) // 2]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tuples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(secs) / len(secs), 3),
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": ws.name, "rows": ws.total_rows, "sample_rows_per_step": budget},
            "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": base["cores"], "kind": "oracle",
                             "sample": base["sample"]},
            "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4", choices=["C1", "C2", "C3", "C3t", "C4", "C5", "C5-cycle"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cpu-rows", type=int, default=300_000_000)
    ap.add_argument("--ref-rows", type=int, default=100_000_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--wire", default="i32", choices=["i32", "i64"], help="all-reduce wire format (N > 1)")
    ap.add_argument("--no-overlap", action="store_true", help="one trailing all-reduce instead of per-table ones")
    ap.add_argument("--row-shard", action="store_true",
                    help="reduce-scatter by sketch row + row-sharded composition instead of the all-reduce (graph workloads)")
    ap.add_argument("--merge", default="nccl", choices=["nccl", "peer"],
                    help="cross-GPU merge: NCCL all-reduce, or pushes over peer memory fused into the scans "
                         "(SURVEY.md 8(f) 4, P2P variant)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args.gpus))
    world, rank, local = _setup_dist()
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            dist.destroy_process_group()
        return
    from paper_2102_02440_b200 import kernel_launches
    from paper_2102_02440_b200.query import QueryRun

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ws = _workload(args.workload, args.scale)
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    data = {t.name: datagen.generate_table(ws, t.name, dev, rank=rank, world=world) for t in ws.tables}
    torch.cuda.synchronize()
    # N > 1: int32 wire and per-table all-reduces overlapped with the next table's scan
    # (SURVEY.md §8(e) levers i and ii); N = 1 has no collective
    run = QueryRun(ws, dev, wire=args.wire, overlap=not args.no_overlap, merge=args.merge)
    subplans = _subplans(ws) if ws.kind == "graph" else None
    stream = torch.cuda.current_stream()
    kev = []  # (start, end) events around each fused-scan launch
    pev = []  # per step: (start, build done = sketches resident after the all-reduce, end)

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def step(record=False):
        s0 = ev() if record else None
        run.zero_(stream)
        for t in ws.tables:
            a = ev() if record else None
            run.build_table(t.name, data[t.name], preds[t.name], stream=stream)
            if record:
                kev.append((a, ev()))
        if args.row_shard and subplans is not None:
            # lever iii: reduce-scatter by sketch row, row-sharded composition, one all-gather
            # of the per-row exact values per greedy level
            shards, own = run.merge_rows()
            s1 = ev() if record else None
            plan = run.plan_greedy_rowshard(shards, own)
            if record:
                pev.append((s0, s1, ev()))
            return None, plan
        run.allreduce()
        s1 = ev() if record else None
        g = run.graph()
        if subplans is None:
            # C4: self-join size of each key sketch, one batched estimate call
            ests = g.estimate_subplans([(g.tables[2 * i], g.tables[2 * i + 1]) for i in range(len(g.tables) // 2)])
            plan = None
        else:
            # plan_greedy evaluates the connected sub-plans it needs (A11), then plans (A12)
            ests = None
            plan = g.plan_greedy()
        if record:
            pev.append((s0, s1, ev()))
        return ests, plan

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier(world)
    l0 = kernel_launches()
    with ClockSampler(local) as clk:
        _barrier(world)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ests, plan = step(record=True)
        e1.record(stream)
        torch.cuda.synchronize()
        _barrier(world)
    launches = kernel_launches() - l0
    if ests is None:
        ests = run.graph().estimate_subplans(subplans)   # for the report only (outside the timed region)
    ms = e0.elapsed_time(e1) / args.steps
    ms = _max_over_ranks(ms, world)
    kms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    kms = _max_over_ranks(kms, world)
    # t_build: first kernel of the step -> final int64 sketches resident
    # (after the all-reduce for N > 1); max over ranks
    bms = _max_over_ranks(sum(a.elapsed_time(b) for a, b, _ in pev) / args.steps, world)
    ems = _max_over_ranks(sum(b.elapsed_time(c) for _, b, c in pev) / args.steps, world)
    rows_all = ws.total_rows
    value = rows_all / (bms / 1e3)

    # roofline of the dominant kernel (the fused scan), algorithmic bytes per launch set
    ab = algorithmic_bytes(ws, data, preds, run)
    peaks = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = ab["alg"] / (kms / 1e3) / 1e9
    traffic = None
    try:
        tf = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tf.get(ws.name)
    except Exception:
        pass
    roofs = _measured_roofs()
    read_peak = roofs.get("read_stream_gbs")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": "k_scan (persistent TMA-ring fused filter+hash+update+flush)",
            "alg_bytes_per_step": ab["alg"], "kernel_ms_per_step": round(kms, 4),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "_fallback" not in peaks else "fallback 6.65 TB/s",
            "frac_of_nominal_8TBs": round(achieved / 8000.0, 4)}
    if read_peak:
        # third denominator of SURVEY.md §8(d): the measured read-only stream (MEASURED_ROOFS.json)
        roof["read_stream_gbs"] = read_peak
        roof["frac_of_read_stream"] = round(achieved / read_peak, 4)
    roof.update(_int_update_roofs(ws, run.survivors.tolist(), kms, roofs))
    br = binding_roof(ws, run.survivors.tolist(), ab["per_table"], kms, peak, roofs)
    if br:
        roof["binding"] = br
    line = {"metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "timing": {"value_is": "rows of all ranks / t_build (SURVEY.md 8(d)): zero + fused scans + "
                                   "all-reduce, max over ranks; every step also runs the estimates and the plan",
                       "build_ms_per_step": round(bms, 4), "estimate_plan_ms_per_step": round(ems, 4),
                       "step_ms": round(ms, 4), "step_tuples_per_s": rows_all / (ms / 1e3)},
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded counter-based generator, datagen/)",
            "config": {"workload": ws.name, "rows": rows_all, "tables": len(ws.tables),
                       "sketches": [f"{s.table}:{'x'.join(map(str, s.w))}xd{s.d}" for s in ws.sketches],
                       "subplans": len(subplans) if subplans else len(ests),
                       "l2": "inputs larger than L2 (no flush)" if ab["full"] > 4 * 126e6 else "inputs L2-resident",
                       "parallelism": f"row-sharded x{world}" + (
                           " + NCCL reduce-scatter by sketch row, row-sharded composition" if (args.row_shard and subplans)
                           else " + pushes over peer memory fused into the scans (CUDA IPC, red.add)" if args.merge == "peer"
                           else (f" + NCCL SUM all-reduce ({run.merge.wire} wire, "
                                 f"{'per-table overlapped' if run.merge.overlap else 'one trailing'})" if world > 1 else ""))},
            "roofline": roof, "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "survivors": run.survivors.tolist(), "estimates": ests[:8] if ests else None,
            "rates": {"survivors_per_s": sum(run.survivors.tolist()) / (bms / 1e3),
                      "row_updates_per_s": sum(surv_n * sum(s.d for s in ws.sketches_of(t.name))
                                               for t, surv_n in zip(ws.tables, run.survivors.tolist())) / (bms / 1e3)},
            "plan": plan[0] if plan else None}

    # end to end through the public API with pinned host buffers (H2D inside the timed region)
    if not args.no_e2e:
        try:
            line["e2e"] = e2e(ws, data, preds, run, subplans, world, stream, args)
        except Exception as ex:  # report, never hide
            line["e2e"] = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_oracle_sample(ws, args.cpu_rows, dev)
        except Exception as ex:
            line["cpu_baseline"] = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
    if world > 1:
        comm = _nccl_comm_line()
        line["nccl"] = {"comm": comm, "world_size": dist.get_world_size()}
        if rank == 0 and comm:
            print(comm, flush=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e(ws, data, preds, run, subplans, world, stream, args, chunk_rows=1 << 26, e2e_steps=2):
    """Same metric, columns streamed from pinned host memory each step: chunked H2D on a
    copy stream overlapped with the fused scans (exact by linearity), then all-reduce,
    estimates and plan read back to the host."""
    host = {}
    for t in ws.tables:
        host[t.name] = {}
        for c, v in data[t.name].items():
            h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
            h.copy_(v)
            host[t.name][c] = h
    cstream = torch.cuda.Stream()
    # tables with predicates: their key columns stay in pinned host memory and the fused scan
    # gathers only the survivors' key sectors over PCIe (zero-copy); predicate columns (and
    # every column of a table without predicates) are copied in chunks
    zc = {}
    for t in ws.tables:
        pcols = {p[0] for p in preds[t.name]}
        zc[t.name] = {c for c in data[t.name] if preds[t.name] and c not in pcols}
    bufs = [{c: torch.empty(min(chunk_rows, v.numel()), dtype=v.dtype, device=v.device)
             for c, v in data[t.name].items() if c not in zc[t.name]}
            for t in ws.tables for _ in range(2)]
    h2d = sum(v.numel() * v.element_size() for t in ws.tables for c, v in data[t.name].items() if c not in zc[t.name])
    ab = algorithmic_bytes(ws, data, preds, run)   # key-column sectors holding a survivor (zero-copy reads)
    h2d_zc = ab["alg"] - run.sketch_bytes - sum(data[t.name][c].numel() * data[t.name][c].element_size()
                                                  for t in ws.tables for c in {p[0] for p in preds[t.name]})

    last_use = {}

    def one_step():
        run.zero_()
        k = 0
        for ti, t in enumerate(ws.tables):
            n = next(iter(host[t.name].values())).numel()
            for s in range(0, n, chunk_rows):
                e = min(n, s + chunk_rows)
                bi = (2 * ti) + (k & 1)
                buf = bufs[bi]
                done = torch.cuda.Event()
                with torch.cuda.stream(cstream):
                    if bi in last_use:            # the scan that last read this staging buffer
                        cstream.wait_event(last_use[bi])
                    for c, hv in host[t.name].items():
                        if c not in zc[t.name]:
                            buf[c][:e - s].copy_(hv[s:e], non_blocking=True)
                    done.record(cstream)
                stream.wait_event(done)
                cols = {c: (host[t.name][c][s:e] if c in zc[t.name] else buf[c][:e - s]) for c in host[t.name]}
                run.build_table(t.name, cols, preds[t.name], stream=stream)
                used = torch.cuda.Event()
                used.record(stream)
                last_use[bi] = used
                k += 1
        run.allreduce()
        g = run.graph()
        if subplans is None:
            ests = g.estimate_subplans([(g.tables[2 * i], g.tables[2 * i + 1]) for i in range(len(g.tables) // 2)])
        else:
            ests = g.plan_greedy()
        return ests

    one_step()
    torch.cuda.synchronize()
    _barrier(world)
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        one_step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / e2e_steps
    ms = _max_over_ranks(ms, world)
    d2h = 8 * (len(ws.tables) + (len(subplans) if subplans else 2))
    return {"value": ws.total_rows / (ms / 1e3), "unit": "tuples/s", "h2d_bytes_per_step": h2d + h2d_zc,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3), "steps": e2e_steps,
            "h2d_copied_bytes": h2d, "h2d_zero_copy_key_sector_bytes": h2d_zc,
            "note": "pinned host columns; predicate columns copied in 64M-row chunks on a copy stream "
                    "overlapped with the fused scan; key columns of filtered tables read in place "
                    "(zero-copy, survivors' sectors only)"}


if __name__ == "__main__":
    main()
