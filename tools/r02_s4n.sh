#!/bin/bash
# current C3 estimate kernels: launch list of the C3 bench step and ncu --set full of k_node_merged_x
O=gpurun_out/s4n; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/c3_launches.csv python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/c3_launches.log 2>&1; echo "list rc=$?"
python tools/ncu_summary.py --launches $O/c3_launches.csv > $O/c3_launches.txt 2>&1; head -20 $O/c3_launches.txt
R=/tmp/ncu_c3mx
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_node_merged_x -s 20 -c 2 -o $R python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_mx.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py $R.ncu-rep > $O/sum_mx.txt 2>&1; head -60 $O/sum_mx.txt
ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 40 > $O/lines_mx.txt 2>&1; head -30 $O/lines_mx.txt
