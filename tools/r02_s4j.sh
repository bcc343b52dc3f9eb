#!/bin/bash
# L2 prefetch size of the survivor-key gathers: .L2::64B (default) vs none vs .L2::128B
O=gpurun_out/s4j; mkdir -p $O
for v in default nohint l2128; do
  if [ $v = default ]; then unset COMPASS_LIB; else export COMPASS_LIB=$PWD/build_var/libcompass_$v.so; fi
  timeout 300 python tools/scan_bench.py --workload C4 --iters 10 > $O/sb_C4_$v.json 2>&1
  timeout 300 python tools/scan_bench.py --workload C5 --iters 5 > $O/sb_C5_$v.json 2>&1
  python -c "
import json
a=json.load(open('$O/sb_C4_$v.json'))['tables']; b=json.load(open('$O/sb_C5_$v.json'))['tables']
print('$v', 'C4', {k: v['ms'] for k, v in a.items()}, 'C5', {k: v['ms'] for k, v in b.items()}, round(sum(v['ms'] for v in b.values()),3))"
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_scan -s 2 -c 1 python tools/scan_bench.py --workload C4 --iters 2 --warmup 1 > $O/ncu_C4_$v.txt 2>&1
  grep -E "dram__bytes_read.sum|gpu__time_duration" $O/ncu_C4_$v.txt | sed "s/^/$v /"
done
