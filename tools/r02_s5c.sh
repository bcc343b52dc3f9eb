#!/bin/bash
# A/B of the unrolled residue mat-vec: C5-cycle / C5 / C3 bench lines, then the GPU suite.
O=gpurun_out/s5c; mkdir -p $O
for w in C5-cycle C5 C3; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_$w.log 2>&1; echo "$w rc=$?"; grep '^{' $O/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'])"; done
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
