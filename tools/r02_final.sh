#!/bin/bash
# Round-2 measurement pass: every bench line, the C4 launch list, the reference arm, the GPU suite.
O=gpurun_out/final; mkdir -p $O
nproc > $O/nproc.txt
python bench.py --steps 10 --warmup 3 > $O/bench_C4.log 2>&1
for w in C1 C2 C3 C3t C5 C5-cycle; do python bench.py --workload $w --steps 5 --warmup 3 --no-e2e > $O/bench_$w.log 2>&1; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_C4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/c4_launches.log 2>&1
python tools/ncu_summary.py --launches $O/c4_launches.csv > $O/c4_launches.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
