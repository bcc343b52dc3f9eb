#!/bin/bash
# knob sweep of the mid-selectivity C5 tables (sub-tiles, TMA stages, key-ring depth)
O=gpurun_out/s4d; mkdir -p $O
timeout 900 python tools/sweep_scan.py --workload C5 --tables T5,T6,T7,T8,T9,T10 > $O/sweep_C5.json 2> $O/sweep_C5.err; echo rc=$?
tail -2 $O/sweep_C5.err
python -c "
import json; d=json.load(open('$O/sweep_C5.json'))
for t, r in d['tables'].items(): print(t, 'default', r['default'], 'best', r['best'], r[r['best']])"
