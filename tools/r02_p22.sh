#!/bin/bash
O=gpurun_out/p22; mkdir -p $O /tmp/ncu
for spec in "C5 T6" "C5 T7"; do
  set -- $spec
  R=/tmp/ncu/ncu_${1}_${2}
  ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 40 > $O/lines_${1}_${2}.txt 2>&1
done
python -m pytest tests/test_multigpu_nccl.py -q > $O/nccl.log 2>&1
tail -3 $O/nccl.log
