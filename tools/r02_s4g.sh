#!/bin/bash
# (1) debug build with device-side bounds checks (-DCOMPASS_CHECKS; compute-sanitizer is closed
#     on the pool) through every k_scan variant and the lookup / histogram / C4 / C5 parity tests;
# (2) ncu --set full of the mid-selectivity C5 scans (T6, T7) and the one-key T10 scan
O=gpurun_out/s4g; mkdir -p $O
export COMPASS_LIB=$PWD/build_var/libcompass_checks.so
timeout 600 python tools/sanitize.py > $O/checks_sanitize.log 2>&1; echo "checks sanitize rc=$?"; tail -3 $O/checks_sanitize.log
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_parity_gpu_extra.py -m gpu -q -x -k "scan or build or fast or lut or hist or kw or ring or c4 or c5 or tensor" > $O/checks_pytest.log 2>&1; echo "checks pytest rc=$?"; tail -2 $O/checks_pytest.log
unset COMPASS_LIB
for spec in "C5 T6" "C5 T7" "C5 T10"; do
  set -- $spec
  R=/tmp/ncu_${1}_${2}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 60 > $O/lines_${1}_${2}.txt 2>&1
  ls -la $R.ncu-rep >> $O/reps.txt
done
