#!/bin/bash
# ncu --set full of the C4 scan and the C5 T9 / T10 scans with the final binary
O=gpurun_out/s4p; mkdir -p $O
for spec in "C4 F" "C5 T9" "C5 T10"; do
  set -- $spec
  R=/tmp/ncu_s4p_${1}_${2}
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1; echo "ncu $1 $2 rc=$?"
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 60 > $O/lines_${1}_${2}.txt 2>&1
  head -3 $O/sum_${1}_${2}.txt
done
