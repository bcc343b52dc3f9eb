"""Per (kernel, grid, block) totals of an ncu --metrics gpu__time_duration.sum --csv launch list,
divided by the number of steps the command ran: python tools/ncu_grid.py launches.csv STEPS"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    key = (r[ix["Kernel Name"]].split("(")[0], r[ix["Grid Size"]], r[ix["Block Size"]])
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    v = v * 1e3 if u == "ms" else (v / 1e3 if u == "ns" else v)
    agg[key][0] += 1
    agg[key][1] += v
tot = sum(t for _, t in agg.values()) or 1
print(f"{'kernel':34s} {'grid':>16s} {'block':>12s} {'launches':>8s} {'us/step':>10s} {'us/launch':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{k[0][:34]:34s} {k[1]:>16s} {k[2]:>12s} {c:8d} {t / steps:10.1f} {t / c:10.1f} {t / tot * 100:6.1f}%")
