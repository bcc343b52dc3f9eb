#!/bin/bash
O=gpurun_out/p26; mkdir -p $O
COMPASS_SCAN_DEBUG=1 timeout 300 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "tensor3_scan" > $O/t.log 2>&1; tail -3 $O/t.log
COMPASS_SCAN_DEBUG=1 COMPASS_LIB=build_var/libcompass_dbg3.so timeout 600 cuda-gdb -batch -ex run -ex bt -ex "info registers rip" --args python tools/c3t_repro.py 0.01 > $O/gdb.log 2>&1; echo "gdb rc=$?"
tail -60 $O/gdb.log
