#!/bin/bash
O=gpurun_out/p38; mkdir -p $O
for v in long __int128; do
ncu --set full --import-source on --clock-control none --kernel-name-base demangled --kernel-name regex:"merged_x<$v>" -c 1 -o /tmp/mx_$v python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
python tools/ncu_summary.py /tmp/mx_$v.ncu-rep > $O/mx_${v}_full.txt 2>&1
ncu -i /tmp/mx_$v.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$v.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_$v.csv 40 > $O/mx_${v}_lines.txt 2>&1
head -25 $O/mx_${v}_full.txt; head -30 $O/mx_${v}_lines.txt
done
