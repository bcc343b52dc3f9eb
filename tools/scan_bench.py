#!/usr/bin/env python
"""Time the fused scan (sketch_update_filtered) of one workload table in isolation.

    python tools/scan_bench.py --workload C4 --table F --scale 0.1 --iters 10 [--generic]

Prints one JSON line: ms per launch (CUDA events on the launching stream, after
warm-up), algorithmic bytes and GB/s.  Used for iteration and as
the command profiled by ncu (profiles/).
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
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--table", default=None)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--generic", action="store_true")
    args = ap.parse_args()
    if args.generic:
        os.environ["COMPASS_SCAN"] = "generic"
    import datagen
    from paper_2102_02440_b200.query import QueryRun
    dev = torch.device("cuda", 0)
    ws = bench._workload(args.workload, args.scale)
    tables = [args.table] if args.table else [t.name for t in ws.tables]
    run = QueryRun(ws, dev)
    out = {"workload": ws.name, "scale": args.scale, "tables": {}}
    for name in tables:
        data = {name: datagen.generate_table(ws, name, dev)}
        preds = {name: datagen.resolve_preds(ws, name)}
        s = torch.cuda.current_stream()
        for _ in range(args.warmup):
            run.build_table(name, data[name], preds[name], stream=s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(args.iters):
            run.build_table(name, data[name], preds[name], stream=s)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        sub = type(ws)(ws.name, [ws.table(name)], [], ws.sketches_of(name), ws.master_seed, ws.data_seed, ws.kind)
        sub_run = type("R", (), {"sketch_bytes": sum(8 * s_.d * (s_.w[0] * (s_.w[1] if len(s_.w) > 1 else 1))
                                                     for s_ in ws.sketches_of(name))})()
        ab = bench.algorithmic_bytes(sub, data, preds, sub_run)
        rows = ws.table(name).n_rows
        out["tables"][name] = {"rows": rows, "ms": round(ms, 4), "alg_bytes": ab["alg"], "full_bytes": ab["full"],
                               "gbs_alg": round(ab["alg"] / ms / 1e6, 1), "rows_per_s": rows / ms * 1e3}
        del data
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
