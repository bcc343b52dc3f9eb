#!/bin/bash
# measured stage / ring rule: per-table scans, bench lines, scan parity
O=gpurun_out/s4f; mkdir -p $O
for w in C5 C5-cycle; do
  timeout 300 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}.json 2>&1
  python -c "
import json; d=json.load(open('$O/sb_${w}.json')); print('$w', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
done
for w in C5 C5-cycle C2 C4; do
timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_$w.log 2>&1
grep '^{' $O/b_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w', t['build_ms_per_step'], t['estimate_plan_ms_per_step'], d['roofline']['frac'])"
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py tests/test_fullsize_gpu.py -m gpu -q -x -k "scan or build or fast or lut or c5 or kw or ring or full" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
