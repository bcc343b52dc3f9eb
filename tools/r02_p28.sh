#!/bin/bash
# full GPU suite after 3-D tensors moved into k_scan; C3t bench line; C4 launch list of our kernels
O=gpurun_out/p28; mkdir -p $O
python bench.py --workload C3t --steps 5 --warmup 3 --no-e2e > $O/bench_C3t.log 2>&1; echo "c3t rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/c4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/c4_launches.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py --launches $O/c4_launches.csv > $O/c4_launches.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
