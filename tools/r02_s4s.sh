#!/bin/bash
# matrix residues shared by the greedy levels of one planning call: C5 / C5-cycle / C2 / C3 estimate
# timings and the estimate parity tests
O=gpurun_out/${S4S_OUT:-s4s}; mkdir -p $O
for w in C5 C5-cycle C2 C3; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$w.log 2>&1
grep '^{' $O/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], d['plan'], d['gpu_launches'])"
done
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py tests/test_fullsize_gpu.py tests/test_multigpu_nccl.py -m gpu -q -x -k "estimate or plan or c5 or c2 or c3 or engine or greedy or enumerate or row" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
