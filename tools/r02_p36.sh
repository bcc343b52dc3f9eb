#!/bin/bash
O=gpurun_out/p36; mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "cycle_gemm" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
timeout 300 python bench.py --workload C5-cycle --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b.log 2>&1
grep '^{' $O/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print(t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'], d['estimates'][:2])"
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'k_node_mat_gemm_bulk|k_planes' --csv --log-file $O/l_gemm.csv python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_gemm.log 2>&1
python tools/ncu_grid.py $O/l_gemm.csv 4 2>/dev/null | head -5
