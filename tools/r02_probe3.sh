#!/bin/bash
O=gpurun_out/pr3
mkdir -p $O /tmp/ncu
tools/mc_probe > $O/mc_probe.txt 2>&1
python -m pytest tests/test_parity_gpu_extra.py -q -x -k "lookup" > $O/extra.log 2>&1
for w in C5 C5-cycle C2; do python tools/scan_bench.py --workload $w --iters 5 > $O/sb_$w.json 2>&1; done
for st in 4 6 8; do COMPASS_STAGES=$st python tools/scan_bench.py --workload C5 --table T2 --iters 5 > $O/sb_T2_st$st.json 2>&1; done
for spec in "C5 T2" "C5 T8"; do
  set -- $spec
  R=/tmp/ncu/ncu_${1}_${2}
  ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 60 > $O/lines_${1}_${2}.txt 2>&1
done
