#!/bin/bash
O=gpurun_out/p34; mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "cycle_gemm" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
for w in C5-cycle C5; do for v in default NO_RES; do
  if [ $v = NO_RES ]; then export COMPASS_EST_NO_RES=1; else unset COMPASS_EST_NO_RES; fi
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_${w}_$v.log 2>&1
  grep '^{' $O/b_${w}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w $v', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'], d['estimates'][:2])"
done; done
unset COMPASS_EST_NO_RES
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'k_node_mat_gemm_bulk|k_planes' --csv --log-file $O/l_gemm.csv python bench.py --workload C5-cycle --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_gemm.log 2>&1
python tools/ncu_grid.py $O/l_gemm.csv 4
