#!/bin/bash
O=gpurun_out/p33; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_c5c.csv python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c5c.log 2>&1; echo "ncu rc=$?"
python tools/ncu_grid.py $O/l_c5c.csv 4 > $O/l_c5c.txt; head -30 $O/l_c5c.txt
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_node_mat_gemm_bulk' -c 1 -o /tmp/gemm_bulk python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_gemm.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/gemm_bulk.ncu-rep > $O/gemm_bulk_full.txt 2>&1
ncu -i /tmp/gemm_bulk.ncu-rep --page raw --csv > $O/gemm_bulk_raw.csv 2>&1
head -30 $O/gemm_bulk_full.txt
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_c3.csv python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c3.log 2>&1; echo "ncu c3 rc=$?"
python tools/ncu_grid.py $O/l_c3.csv 4 > $O/l_c3.txt; head -30 $O/l_c3.txt
