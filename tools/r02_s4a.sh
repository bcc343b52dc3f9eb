#!/bin/bash
# Session-4 baseline on the current HEAD: smoke, GPU suite, bench lines C4 / C5 / C5-cycle / C3.
O=gpurun_out/s4a; mkdir -p $O
nvidia-smi -L > $O/gpu.txt 2>&1; nproc >> $O/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_C4.log 2>&1; echo "c4 rc=$?"
for w in C5 C5-cycle C3; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_$w.log 2>&1; echo "$w rc=$?"; done
for w in C4 C5 C5-cycle C3; do grep '^{' $O/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', d['value'], t.get('build_ms_per_step'), t.get('estimate_plan_ms_per_step'), d['roofline']['frac'])"; done
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
