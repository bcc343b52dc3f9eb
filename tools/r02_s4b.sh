#!/bin/bash
# Two-stream overlap of the C5 scans with disjoint CTA budgets (tools/overlap_bench.py)
O=gpurun_out/s4b; mkdir -p $O
for w in C5 C5-cycle; do timeout 600 python tools/overlap_bench.py --workload $w --iters 5 > $O/ov_$w.json 2>$O/ov_$w.err; echo "$w rc=$?"; tail -3 $O/ov_$w.err; cat $O/ov_$w.json; done
