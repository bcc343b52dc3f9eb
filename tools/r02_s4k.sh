#!/bin/bash
# 1-D lookup-table updates as red.shared at 32-bit shared addresses, d = 5 unrolled without bound checks
O=gpurun_out/s4k; mkdir -p $O
for w in C5 C5-cycle C2 C3; do
  timeout 300 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}.json 2>&1
  python -c "
import json; d=json.load(open('$O/sb_${w}.json')); print('$w', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
done
timeout 300 python tools/scan_bench.py --workload C4 --iters 10 > $O/sb_C4.json 2>&1; cat $O/sb_C4.json | head -c 300; echo
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x -k "scan or build or fast or lut or c5 or kw or ring or hist or c2 or c3" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
