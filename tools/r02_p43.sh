#!/bin/bash
O=gpurun_out/p43; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x -k "c5 or cycle or random or row_shard" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
for w in C5 C5-cycle; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$w.log 2>&1
grep '^{' $O/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'k_mat_residues|k_node_matvec_r' --csv --log-file $O/l_c5.csv python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_c5.log 2>&1
python tools/ncu_grid.py $O/l_c5.csv 4 2>/dev/null | head -6
