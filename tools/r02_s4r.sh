#!/bin/bash
# launch lists of the C5-cycle and C5-chain steps (own kernels), for the estimate-side breakdown
O=gpurun_out/s4r; mkdir -p $O
for w in C5-cycle C5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_$w.log 2>&1; echo "list $w rc=$?"
python tools/ncu_summary.py --launches $O/l_$w.csv > $O/l_$w.txt 2>&1; head -16 $O/l_$w.txt
done
