#!/bin/bash
# C5 per-table scan variants + ncu captures of the slow tables (round-2 probe)
set -x
O=gpurun_out/c5p
mkdir -p $O
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
  ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $O/ncu_${1}_${2} python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1
done
