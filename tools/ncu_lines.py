#!/usr/bin/env python
"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line.

    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows, fname, hdr = [], None, None
    with open(path) as f:
        for rec in csv.reader(f):
            if not rec:
                continue
            if rec[0] == "File Path":
                fname = rec[1].split("/")[-1]
                continue
            if rec[0] == "Line No":
                hdr = rec
                continue
            if hdr is None or rec[0] in ("", "Function Name"):
                continue
            d = dict(zip(hdr[2:], rec[2:]))  # skip duplicated 'Source' key collisions
            try:
                inst = int(rec[hdr.index("Instructions Executed")])
                samp = int(rec[hdr.index("Warp Stall Sampling (All Samples)")])
            except (ValueError, IndexError):
                continue
            rows.append((inst, samp, f"{fname}:{rec[0]}", rec[1][:90]))
    tot_i = sum(r[0] for r in rows) or 1
    tot_s = sum(r[1] for r in rows) or 1
    print(f"total warp-instructions {tot_i:,}  samples {tot_s:,}")
    for inst, samp, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{inst / tot_i * 100:6.2f}% inst {samp / tot_s * 100:6.2f}% samp  {loc:18s} {src}")


if __name__ == "__main__":
    main()
