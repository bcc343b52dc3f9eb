#!/bin/bash
# ncu --set full of the C5-cycle step's top estimation kernels (k_node_matvec_r, k_mat_residues)
O=gpurun_out/s5b; mkdir -p $O
for k in k_node_matvec_r k_mat_residues; do
  R=/tmp/ncu_$k
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"^$k" -s 40 -c 1 -o $R python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_$k.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 40 > $O/lines_$k.txt 2>&1
done
