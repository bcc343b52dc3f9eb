"""Build C3t table by table at a small scale, printing progress (crash localisation)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2102_02440_b200.query import QueryRun

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
ws = datagen.c3t(scale=scale)
dev = torch.device("cuda", 0)
run = QueryRun(ws, dev)
for t in ws.tables:
    dd = datagen.generate_table(ws, t.name, dev)
    print("table", t.name, t.n_rows, [s.key_cols for s in ws.sketches_of(t.name)], flush=True)
    run.build_table(t.name, dd, datagen.resolve_preds(ws, t.name))
    torch.cuda.synchronize()
    print("  ok", flush=True)
