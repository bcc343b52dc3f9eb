#!/bin/bash
# survivor-ring depth: adaptive (default) vs fixed caps on the C5 / C5-cycle tables
O=gpurun_out/p48; mkdir -p $O
for w in C5 C5-cycle; do
for cap in def 64 128 256 512 1024; do
  if [ $cap = def ]; then unset COMPASS_CAP; else export COMPASS_CAP=$cap; fi
  timeout 300 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}_$cap.json 2>&1
  python -c "
import json; d=json.load(open('$O/sb_${w}_$cap.json')); print('$w cap $cap', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
done
done
unset COMPASS_CAP
COMPASS_SCAN_DEBUG=1 timeout 300 python tools/scan_bench.py --workload C5 --iters 1 --warmup 1 2>&1 | grep 'k_scan plan' | sort | uniq > $O/plans_C5.txt
cat $O/plans_C5.txt
timeout 300 python bench.py --workload C4 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_C4.log 2>&1
grep '^{' $O/b_C4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('C4', t['build_ms_per_step'], d['roofline']['frac'])"
