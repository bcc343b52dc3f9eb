#!/bin/bash
O=gpurun_out/p27; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "tensor3 or c3t or lookup or hist" > $O/t.log 2>&1; tail -3 $O/t.log
COMPASS_SCAN_DEBUG=1 COMPASS_LIB=build_var/libcompass_checked.so timeout 300 python tools/c3t_repro.py 0.1 > $O/chk.log 2>&1; echo "checked rc=$?"; tail -5 $O/chk.log
COMPASS_SCAN_DEBUG=1 timeout 300 python bench.py --workload C3t --steps 5 --warmup 3 --no-e2e > $O/c3t.log 2>&1; echo "opt rc=$?"
grep "k_scan" $O/c3t.log | sort | uniq -c | head; tail -c 1500 $O/c3t.log
