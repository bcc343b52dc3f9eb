#!/bin/bash
O=gpurun_out/p15; mkdir -p $O
python -m pytest tests/test_parity_gpu_extra.py -q -x -k "lookup" > $O/t_lookup.log 2>&1
for w in C5 C5-cycle C2; do
  python tools/scan_bench.py --workload $w --iters 5 > $O/sb_$w.json 2>&1
  COMPASS_BIN=0 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}_nobin.json 2>&1
done
python bench.py --workload C3 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c3.log 2>&1
python -m pytest tests/test_parity_gpu.py -q -x -k "estimates or c3 or c5 or c2 or c1 or accuracy" > $O/t_est.log 2>&1
tail -2 $O/t_lookup.log $O/t_est.log
