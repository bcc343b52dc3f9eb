#!/usr/bin/env python
"""Decompose the C4 fused-scan time: pure predicate streaming vs survivor gathers vs updates."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2102_02440_b200 as pb  # noqa: E402


def timeit(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    dev = torch.device("cuda", 0)
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    ws = datagen.c4(scale=scale)
    t = ws.tables[0]
    data = datagen.generate_table(ws, "F", dev)
    names = [c.name for c in t.cols]
    cols = [data[c] for c in names]
    n = cols[0].numel()
    s1 = pb.Sketch(9, [16384], [ws.sketches[0].edge_ids[0]], 42, dev)
    s2 = pb.Sketch(9, [16384], [ws.sketches[1].edge_ids[0]], 42, dev)
    real = [(names.index(f"p{i}"), pb.RANGE, pb.INT64_MIN, 367) for i in (1, 2, 3)]
    none = [(names.index(f"p{i}"), pb.RANGE, pb.INT64_MIN, -1) for i in (1, 2, 3)]
    k1, k2 = names.index("key1"), names.index("key2")
    out = {}
    out["stream_3pred_no_survivor_ms"] = timeit(lambda: pb.sketch_update_filtered(cols, n, none, [(s1, [k1]), (s2, [k2])]))
    out["real_1key_ms"] = timeit(lambda: pb.sketch_update_filtered(cols, n, real, [(s1, [k1])]))
    out["real_2key_ms"] = timeit(lambda: pb.sketch_update_filtered(cols, n, real, [(s1, [k1]), (s2, [k2])]))
    out["real_1pred_2key_ms"] = timeit(lambda: pb.sketch_update_filtered(cols, n, real[:1], [(s1, [k1]), (s2, [k2])]))
    out["copy_12GB_ms"] = timeit(lambda: torch.cat([cols[names.index(f"p{i}")] for i in (1, 2, 3)]).sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
