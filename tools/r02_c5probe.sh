#!/bin/bash
# C5 per-table scan variants + ncu captures of the slow tables (round-2 probe)
O=gpurun_out/c5p
mkdir -p $O /tmp/ncu
for tb in T8 T9 T10; do
  for v in default HIST=0 HISTHH=0 LUT=0; do
    env_args=""
    [ "$v" != default ] && env_args="COMPASS_$v"
    for w in C5 C5-cycle; do
      env $env_args python tools/scan_bench.py --workload $w --table $tb --iters 5 > $O/sb_${w}_${tb}_${v}.json 2>&1
    done
  done
done
for spec in "C5 T9" "C5 T10" "C5-cycle T10" "C5 T8"; do
  set -- $spec
  R=/tmp/ncu/ncu_${1}_${2}
  ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin > $O/lines_${1}_${2}.txt 2>&1
done
du -sh $O
