#!/bin/bash
O=gpurun_out/p14; mkdir -p $O /tmp/ncu
R=/tmp/ncu/c3mx
ncu --set full --clock-control none --import-source on -k regex:k_node_merged_x -s 4 -c 2 -o $R python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu.log 2>&1
python tools/ncu_summary.py $R.ncu-rep > $O/sum_c3mx.txt 2>&1
ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 50 > $O/lines_c3mx.txt 2>&1
ncu -i $R.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:]:
  d=dict(zip(h,r)); print(d.get('Kernel Name','')[:60], d.get('launch__grid_size'), d.get('launch__occupancy_limit_shared_mem'), d.get('sm__warps_active.avg.pct_of_peak_sustained_active'), d.get('launch__shared_mem_per_block_dynamic'))
" > $O/occ.txt 2>&1
