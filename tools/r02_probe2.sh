#!/bin/bash
# ncu of the lookup-table scan on C5 T8/T9/T10 and of C3's estimate kernels
O=gpurun_out/pr2
mkdir -p $O /tmp/ncu
for spec in "C5 T10" "C5 T9" "C5 T8" "C5-cycle T10"; do
  set -- $spec
  R=/tmp/ncu/ncu_${1}_${2}
  ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 60 > $O/lines_${1}_${2}.txt 2>&1
done
# C3 estimation: launch list of one bench step and a full capture of the top merged-node kernel
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_c3.csv python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/l_c3.log 2>&1
R=/tmp/ncu/c3m
ncu --set full --clock-control none --import-source on -k regex:k_node_merged_x -s 6 -c 2 -o $R python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_c3m.log 2>&1
python tools/ncu_summary.py $R.ncu-rep > $O/sum_c3m.txt 2>&1
ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 60 > $O/lines_c3m.txt 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2102_02440_b200/csrc -o /tmp/roofs_micro tools/roofs_micro.cu && /tmp/roofs_micro > $O/roofs.json 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mc_probe tools/mc_probe.cu -lcuda && /tmp/mc_probe > $O/mc_probe.txt 2>&1
nproc > $O/nproc.txt
du -sh $O
