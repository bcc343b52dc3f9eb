#!/bin/bash
O=gpurun_out/p37; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "c3 or random or merged or cycle" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
for i in 1 2; do
timeout 300 python bench.py --workload C3 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_c3_$i.log 2>&1
grep '^{' $O/b_c3_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('C3', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'], d['estimates'][:2])"
done
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_c3.csv python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c3.log 2>&1
python tools/ncu_grid.py $O/l_c3.csv 4 2>/dev/null | head -8
