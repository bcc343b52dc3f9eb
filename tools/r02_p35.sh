#!/bin/bash
O=gpurun_out/p35; mkdir -p $O
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
for w in C5-cycle C5; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$w.log 2>&1
  grep '^{' $O/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'], d['estimates'][:2])"
done
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_c5c.csv python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c5c.log 2>&1
python tools/ncu_grid.py $O/l_c5c.csv 4 | head -24
