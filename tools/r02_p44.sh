#!/bin/bash
# Full GPU suite + bench lines of the current tree (state check at the start of the session)
O=gpurun_out/p44; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for w in C4 C5 C5-cycle C3; do
timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$w.log 2>&1
grep '^{' $O/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'], d['roofline']['frac'])"
done
