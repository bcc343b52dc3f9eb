#!/bin/bash
# ncu captures of the current estimate kernels: tcgen05 cycle GEMM (C5-cycle), exact merged contraction (C3)
O=gpurun_out/p39; mkdir -p $O
ncu --set full --import-source on --clock-control none --kernel-name regex:'k_node_mat_gemm_bulk' -c 1 -o /tmp/gb python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_gb.log 2>&1; echo "gb rc=$?"
python tools/ncu_summary.py /tmp/gb.ncu-rep > $O/gemm_tc_full.txt 2>&1
ncu -i /tmp/gb.ncu-rep --page raw --csv > $O/gemm_tc_raw.csv 2>&1
ncu -i /tmp/gb.ncu-rep --page source --csv --print-source cuda,sass > /tmp/gb_src.csv 2>/dev/null; python tools/ncu_lines.py /tmp/gb_src.csv 30 > $O/gemm_tc_lines.txt 2>&1
for v in long __int128; do
ncu --set full --import-source on --clock-control none --kernel-name-base demangled --kernel-name regex:"merged_x<$v>" --launch-skip 2 -c 1 -o /tmp/mx_$v python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
python tools/ncu_summary.py /tmp/mx_$v.ncu-rep > $O/mx_${v}_full.txt 2>&1
ncu -i /tmp/mx_$v.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$v.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_$v.csv 30 > $O/mx_${v}_lines.txt 2>&1
done
head -25 $O/gemm_tc_full.txt; head -6 $O/mx_long_full.txt; head -22 $O/mx_long_lines.txt; head -6 $O/mx___int128_full.txt; head -22 $O/mx___int128_lines.txt
