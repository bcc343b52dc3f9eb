#!/bin/bash
# C5-cycle step launch list (our kernels only) + ncu full of the TC GEMM
O=gpurun_out/p30; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_c5c.csv python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c5c.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py --launches $O/l_c5c.csv > $O/l_c5c.txt 2>&1
head -30 $O/l_c5c.txt
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_node_mat_gemm_tc' -c 2 -o /tmp/gemm_tc python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_gemm.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/gemm_tc.ncu-rep > $O/gemm_tc_full.txt 2>&1
python tools/ncu_lines.py /tmp/gemm_tc.ncu-rep > $O/gemm_tc_lines.txt 2>&1
head -50 $O/gemm_tc_full.txt
