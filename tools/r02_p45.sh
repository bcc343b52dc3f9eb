#!/bin/bash
# C4 scan after compiling the 3-D tensor drain only into NK >= 3 instances; staged keys A/B on C5
O=gpurun_out/p45; mkdir -p $O
timeout 300 python bench.py --workload C4 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_C4.log 2>&1
grep '^{' $O/b_C4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('C4', t['build_ms_per_step'], d['roofline']['frac'])"
for ks in 0 1; do
COMPASS_KSTAGE=$ks timeout 300 python tools/scan_bench.py --workload C5 --iters 5 > $O/sb_C5_k$ks.json 2>&1
python -c "
import json; d=json.load(open('$O/sb_C5_k$ks.json')); print('kstage $ks', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x -k "scan or build or fast or lut or c4 or c5 or kw or hist or c3t or tensor" > $O/t.log 2>&1; echo "t rc=$?"; tail -2 $O/t.log
COMPASS_KSTAGE=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x -k "scan or build or fast or lut or c5" > $O/t_k1.log 2>&1; echo "t_k1 rc=$?"; tail -2 $O/t_k1.log
