#!/bin/bash
# bulk-fed tensor-core GEMM: parity, then C5-cycle A/B (bulk vs register-fed vs CUDA cores)
O=gpurun_out/p32; mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "cycle_gemm" > $O/t.log 2>&1; echo "t rc=$?"; tail -15 $O/t.log
for g in bulk tc cuda; do
  COMPASS_GEMM=$g timeout 300 python bench.py --workload C5-cycle --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$g.log 2>&1
  grep '^{' $O/b_$g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$g', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], t['step_ms'], d['estimates'][:2])"
done
