#!/usr/bin/env python
"""Sweep the scan's experiment knobs (COMPASS_SUB / COMPASS_STAGES / COMPASS_CAP) per table.

    python tools/sweep_scan.py --workload C5 --tables T5,T6,T7,T8 --iters 8

Each table is generated once; every knob setting is timed with CUDA events on the launching
stream after two warm-up calls, and its counters are compared with the default setting's
(bit-exact: the knobs change scheduling, never results).  One JSON line.
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

KNOBS = ("COMPASS_SUB", "COMPASS_STAGES", "COMPASS_CAP")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--tables", default="T5,T6,T7,T8")
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--sub", default="1,4")
    ap.add_argument("--stages", default="3,4,6,8")
    ap.add_argument("--cap", default="64,128,256")
    args = ap.parse_args()
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    dev = torch.device("cuda", 0)
    ws = bench._workload(args.workload, 1.0)
    run = QueryRun(ws, dev)
    s = torch.cuda.current_stream()
    grid = list(itertools.product(args.sub.split(","), args.stages.split(","), args.cap.split(",")))
    out = {"workload": ws.name, "tables": {}}
    for name in args.tables.split(","):
        data = datagen.generate_table(ws, name, dev)
        preds = datagen.resolve_preds(ws, name)
        mine = [sk for sp, sk in zip(ws.sketches, run.sketches) if sp.table == name]

        def once():
            for sk in mine:
                sk.counters.zero_()
            run.build_table(name, data, preds, stream=s)
            torch.cuda.synchronize()
            return [sk.counters.clone() for sk in mine]

        def timed():
            for _ in range(2):
                run.build_table(name, data, preds, stream=s)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(args.iters):
                run.build_table(name, data, preds, stream=s)
            b.record(s)
            torch.cuda.synchronize()
            return round(a.elapsed_time(b) / args.iters, 4)

        for k in KNOBS:
            os.environ.pop(k, None)
        ref = once()
        res = {"default": timed()}
        for sub, st, cap in grid:
            os.environ.update({"COMPASS_SUB": sub, "COMPASS_STAGES": st, "COMPASS_CAP": cap})
            same = all(torch.equal(x, y) for x, y in zip(ref, once()))
            res[f"sub{sub}_st{st}_cap{cap}"] = timed() if same else "MISMATCH"
        for k in KNOBS:
            os.environ.pop(k, None)
        best = min((v, k) for k, v in res.items() if isinstance(v, float))
        res["best"] = best[1]
        out["tables"][name] = res
        del data
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
