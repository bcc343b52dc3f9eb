#!/usr/bin/env python
"""Accuracy of the sketch estimates on a workload.

    python tools/accuracy.py --workload C2 [--scale 1.0]

Builds the workload's sketches (fused scan), estimates every acyclic connected sub-plan
(estimate_subplans), computes its exact cardinality on the device (exact_join_size) and
prints one JSON line per sub-plan size: median / min / max accuracy ratio (est / true) and
the normalised L1 distance between the estimate order and the true order.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import datagen  # noqa: E402
import evaluation as accuracy  # noqa: E402
from paper_2102_02440_b200.query import QueryRun  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ws = bench._workload(args.workload, args.scale)
    run = QueryRun(ws, dev)
    data = {t.name: datagen.generate_table(ws, t.name, dev) for t in ws.tables}
    preds = {t.name: datagen.resolve_preds(ws, t.name) for t in ws.tables}
    run.build(data, preds)
    torch.cuda.synchronize()
    tables, edges, names = accuracy.join_data(ws, data, preds)
    subs = accuracy.connected_subplans(names, edges)
    t0 = time.perf_counter()
    truths = accuracy.exact_counts(tables, edges, names, subs)
    t_exact = time.perf_counter() - t0
    ests = dict(zip(subs, run.graph().estimate_subplans(subs)))
    rep = accuracy.report(ests, truths)
    for size, (ratios, l1) in rep.items():
        fin = [r for r in ratios if r != float("inf")]
        print(json.dumps({"workload": ws.name, "scale": args.scale, "subplan_tables": size, "subplans": len(ratios),
                          "ratio_median": statistics.median(fin) if fin else None,
                          "ratio_min": min(fin) if fin else None, "ratio_max": max(fin) if fin else None,
                          "l1_normalised": l1, "exact_ms_total": round(t_exact * 1e3, 1),
                          "no_truth": [list(s) for s, v in truths.items() if v is None and len(s) == size]}))


if __name__ == "__main__":
    main()
