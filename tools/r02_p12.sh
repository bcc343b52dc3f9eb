#!/bin/bash
O=gpurun_out/p12; mkdir -p $O
for w in C4 C5 C5-cycle; do python tools/scan_bench.py --workload $w --iters 5 > $O/sb_$w.json 2>&1; done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > $O/sanitizer_$tool.txt 2>&1; echo "exit=$?" >> $O/sanitizer_$tool.txt
done
python -m pytest tests/test_parity_gpu_extra.py tests/test_parity_gpu.py -q -x -k "not full_size" > $O/tests.log 2>&1
tail -2 $O/tests.log
