#!/usr/bin/env python
"""Experiment: do the scans of one query overlap when split over two streams with
disjoint SM budgets?  Tables whose scan is HBM-bound (very selective predicates) run on
stream B with `--ctas-b` CTAs while the issue-bound ones run on stream A with the rest.

    python tools/overlap_bench.py --workload C5 --iters 5

Prints one JSON line per configuration: ms for the whole build (CUDA events on the
default stream, which waits for both), sequential vs split.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--split", type=int, default=5, help="tables [0, split) go to stream B")
    args = ap.parse_args()
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    dev = torch.device("cuda", 0)
    ws = bench._workload(args.workload, 1.0)
    run = QueryRun(ws, dev)
    names = [t.name for t in ws.tables]
    data = {n: datagen.generate_table(ws, n, dev) for n in names}
    preds = {n: datagen.resolve_preds(ws, n) for n in names}
    main_s = torch.cuda.current_stream()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    sms = torch.cuda.get_device_properties(0).multi_processor_count

    def build(cb, order_b, order_a):
        if cb is None:
            os.environ.pop("COMPASS_SCAN_CTAS", None)
            for n in names:
                run.build_table(n, data[n], preds[n], stream=main_s)
            return
        e0 = torch.cuda.Event()
        e0.record(main_s)
        sa.wait_event(e0)
        sb.wait_event(e0)
        ib = ia = 0
        while ib < len(order_b) or ia < len(order_a):   # interleave the enqueues
            if ib < len(order_b):
                os.environ["COMPASS_SCAN_CTAS"] = str(cb)
                n = order_b[ib]; ib += 1
                run.build_table(n, data[n], preds[n], stream=sb)
            if ia < len(order_a):
                os.environ["COMPASS_SCAN_CTAS"] = str(sms - cb)
                n = order_a[ia]; ia += 1
                run.build_table(n, data[n], preds[n], stream=sa)
        os.environ.pop("COMPASS_SCAN_CTAS", None)
        ea, eb = torch.cuda.Event(), torch.cuda.Event()
        ea.record(sa); eb.record(sb)
        main_s.wait_event(ea); main_s.wait_event(eb)

    def timeit(cb, ob, oa):
        for _ in range(2):
            build(cb, ob, oa)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        for _ in range(args.iters):
            build(cb, ob, oa)
        b.record(main_s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.iters

    def snapshot():
        return [sk.counters.clone() for sk in run.sketches]

    # correctness: one build each way from zero, compare counters
    for sk in run.sketches:
        sk.counters.zero_()
    build(None, [], [])
    torch.cuda.synchronize()
    ref = snapshot()
    out = {"workload": ws.name, "sms": sms, "seq_ms": round(timeit(None, [], []), 4), "split": []}
    ob, oa = names[:args.split], names[args.split:][::-1]
    for cb in (16, 24, 32, 48, 64, 74):
        for sk in run.sketches:
            sk.counters.zero_()
        build(cb, ob, oa)
        torch.cuda.synchronize()
        same = all(torch.equal(x, y.counters) for x, y in zip(ref, run.sketches))
        out["split"].append({"ctas_b": cb, "ms": round(timeit(cb, ob, oa), 4), "same": same})
    # per-table at full grid and at reduced grids
    per = {}
    for n in names:
        row = {}
        for cb in (None, 32, 74, 116):
            if cb is None:
                os.environ.pop("COMPASS_SCAN_CTAS", None)
            else:
                os.environ["COMPASS_SCAN_CTAS"] = str(cb)
            for _ in range(2):
                run.build_table(n, data[n], preds[n], stream=main_s)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            for _ in range(args.iters):
                run.build_table(n, data[n], preds[n], stream=main_s)
            b.record(main_s)
            torch.cuda.synchronize()
            row[str(cb or sms)] = round(a.elapsed_time(b) / args.iters, 4)
        per[n] = row
    os.environ.pop("COMPASS_SCAN_CTAS", None)
    out["per_table"] = per
    print(json.dumps(out))


if __name__ == "__main__":
    main()
