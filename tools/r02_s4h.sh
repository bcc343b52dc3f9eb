#!/bin/bash
# sparse per-lane survivor gathers: per-table scans (C5, C5-cycle, C2, C3 tables), C4 bench, scan parity
O=gpurun_out/s4h; mkdir -p $O
for w in C5 C5-cycle C2 C3; do
  timeout 300 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}.json 2>&1
  python -c "
import json; d=json.load(open('$O/sb_${w}.json')); print('$w', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $O/b_C4.log 2>&1
grep '^{' $O/b_C4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('C4', t['build_ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac'])"
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py tests/test_fullsize_gpu.py -m gpu -q -x -k "scan or build or fast or lut or c5 or kw or ring or full or hist" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
