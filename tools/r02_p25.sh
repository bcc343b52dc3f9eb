#!/bin/bash
# 3-D tensors in k_scan: tests, then the C3t crash probe (checked build, faulthandler)
O=gpurun_out/p25; mkdir -p $O
python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "tensor3 or c3t" > $O/t.log 2>&1; tail -3 $O/t.log
for sc in 0.01 0.1 1.0; do
  COMPASS_SCAN_DEBUG=1 COMPASS_LIB=build_var/libcompass_checked.so timeout 300 python -X faulthandler bench.py --workload C3t --scale $sc --steps 2 --warmup 3 --no-e2e --no-cpu > $O/c3t_chk_$sc.log 2>&1; echo "checked $sc rc=$?"
done
COMPASS_SCAN_DEBUG=1 timeout 300 python -X faulthandler bench.py --workload C3t --steps 5 --warmup 3 --no-e2e > $O/c3t.log 2>&1; echo "opt rc=$?"
tail -c 1200 $O/c3t.log
