#!/usr/bin/env python
"""Per-SASS-instruction view of an ncu source page (--print-source cuda,sass --csv):
instructions executed per unit (e.g. per warp-tile) and stall samples, in address order.

    python tools/ncu_sass.py src.csv UNITS [min_per_unit]
"""
import csv
import sys


def main():
    path, units = sys.argv[1], float(sys.argv[2])
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
    hdr, rows = None, []
    for rec in csv.reader(open(path)):
        if rec and rec[0] == "Line No":
            hdr = rec
            continue
        if not rec or hdr is None or rec[0] != "" or len(rec) < 4 or not rec[2].startswith("0x"):
            continue
        try:
            n = int(rec[hdr.index("Instructions Executed")])
            smp = int(rec[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        stalls = {h: rec[i] for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
        top = sorted(((int(v), k[6:]) for k, v in stalls.items() if v.isdigit() and int(v) > 0), reverse=True)[:2]
        rows.append((int(rec[2], 16), rec[3].strip(), n, smp, top))
    rows.sort()
    tot = sum(r[3] for r in rows) or 1
    for a, src, n, smp, top in rows:
        if n / units >= thr or smp / tot > 0.003:
            print(f"{n / units:6.2f} {smp / tot * 100:5.2f}% {src[:60]:60s} {top}")


if __name__ == "__main__":
    main()
