#!/bin/bash
# T3 instances (3-D tensor drain only where a tensor target exists): C4 / C3 / C3t / C2 builds, scan parity
O=gpurun_out/p46; mkdir -p $O
for w in C4 C3 C3t C2; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$w.log 2>&1
grep '^{' $O/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], d['roofline']['frac'])"
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py tests/test_fullsize_gpu.py -m gpu -q -x -k "scan or build or fast or lut or c4 or c5 or kw or hist or c3t or tensor or c3" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
