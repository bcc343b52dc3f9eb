#!/bin/bash
O=gpurun_out/p42; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_c5.csv python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c5.log 2>&1
python tools/ncu_grid.py $O/l_c5.csv 4 2>/dev/null | head -24
