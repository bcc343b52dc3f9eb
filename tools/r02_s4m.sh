#!/bin/bash
# consumer-warp / ring-group configurations (register budget per thread): 20x4 (default, 80
# regs), 16 warps x 4 groups (640 threads, up to 96 regs), 20 warps x 2 groups (704 threads, 88)
O=gpurun_out/s4m; mkdir -p $O
for v in default w16g4 w20g2; do
  if [ $v = default ]; then unset COMPASS_LIB; else export COMPASS_LIB=$PWD/build_var/libcompass_$v.so; fi
  for w in C4 C5 C5-cycle; do
    timeout 300 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}_$v.json 2>&1
    python -c "
import json; d=json.load(open('$O/sb_${w}_$v.json')); print('$v $w', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
  done
done
