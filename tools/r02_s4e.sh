#!/bin/bash
# knob sweep of the C5-cycle tables with two key columns at high selectivity
O=gpurun_out/s4e; mkdir -p $O
timeout 900 python tools/sweep_scan.py --workload C5-cycle --tables T8,T9,T10 --sub 1 --stages 2,3,4,6 --cap 64,128,256,512 > $O/sweep.json 2> $O/sweep.err; echo rc=$?
tail -2 $O/sweep.err
python -c "
import json; d=json.load(open('$O/sweep.json'))
for t, r in d['tables'].items(): print(t, ' '.join(f'{k}={v}' for k,v in r.items()))"
