#!/bin/bash
# staged keys (SK) on the lookup-table path: per-table scans with SK off / auto / forced, parity
O=gpurun_out/s4q; mkdir -p $O
for v in off auto on; do
  if [ $v = off ]; then export COMPASS_SK=0; elif [ $v = on ]; then export COMPASS_SK=1; else unset COMPASS_SK; fi
  for w in C5 C5-cycle C2; do
    timeout 300 python tools/scan_bench.py --workload $w --iters 5 > $O/sb_${w}_$v.json 2>&1
    python -c "
import json; d=json.load(open('$O/sb_${w}_$v.json')); print('$v $w', {k: v['ms'] for k, v in d['tables'].items()}, round(sum(v['ms'] for v in d['tables'].values()),3))"
  done
done
unset COMPASS_SK
COMPASS_SK=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x -k "fast or lut or c5 or c2 or zero" > $O/t_on.log 2>&1; echo "t sk=1 rc=$?"; tail -2 $O/t_on.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py tests/test_peer_merge_gpu.py -m gpu -q -x -k "fast or lut or c5 or c2 or zero or peer" > $O/t_auto.log 2>&1; echo "t auto rc=$?"; tail -2 $O/t_auto.log
