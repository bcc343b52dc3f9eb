#!/usr/bin/env python
"""Summarise an ncu report (--set full) or an ncu launch list (CSV) into text for profiles/.

    python tools/ncu_summary.py report.ncu-rep > profiles/rNN_xxx.txt
    python tools/ncu_summary.py --launches launches.csv > profiles/rNN_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_red.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "smsp__sass_inst_executed_op_shared_atom.sum"]


def ncu_csv(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def report(path):
    rows = list(csv.reader(io.StringIO(ncu_csv(["-i", path, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        print(f"kernel: {d.get('Kernel Name', ('?', ''))[0]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k][0]:>20s} {d[k][1]}")
        stalls = [(h, float(v.replace(',', ''))) for h, v in zip(hdr, vals)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                  and v.replace(',', '').replace('.', '').isdigit()]
        tot = sum(v for _, v in stalls) or 1
        print("  warp-stall samples (share):")
        for h, v in sorted(stalls, key=lambda x: -x[1])[:10]:
            print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v / tot * 100:5.1f}%")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        u = r[ix["Metric Unit"]]
        v = v * 1e3 if u == "ms" else (v / 1e3 if u == "ns" else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values()) or 1
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:60]:60s} {c:8d} {t:12.1f} {t / tot * 100:6.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
