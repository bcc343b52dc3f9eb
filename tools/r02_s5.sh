#!/bin/bash
# Round-2 measurement pass (session 5, head with owner-mode peer merge): smoke, every bench line, peer-merge lines, the reference
# arm, the C4 launch list, ncu --set full of the C4 scan and the C5 T9 scan, the GPU suite.
O=gpurun_out/s5; mkdir -p $O
nproc > $O/nproc.txt; nvidia-smi -L >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_C4.log 2>&1; echo "C4 rc=$?"
for w in C1 C2 C3 C3t C5 C5-cycle; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e > $O/bench_$w.log 2>&1; echo "$w rc=$?"; done
for w in C4 C5; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --merge peer > $O/bench_${w}_peer.log 2>&1; echo "$w peer rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_C4.log 2>&1; echo "ref rc=$?"
for f in $O/bench_*.log; do grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; r=d['roofline']; print('$(basename $f)', round(d['value']/1e9,2), t['build_ms_per_step'], t['estimate_plan_ms_per_step'], r['frac'], (r.get('binding') or {}).get('frac'), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/c4_launches.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py --launches $O/c4_launches.csv > $O/c4_launches.txt 2>&1
for spec in "C4 F" "C5 T9"; do
  set -- $spec
  R=/tmp/ncu_${1}_${2}
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o $R python tools/scan_bench.py --workload $1 --table $2 --iters 2 --warmup 1 > $O/ncu_${1}_${2}.log 2>&1; echo "ncu $1 $2 rc=$?"
  python tools/ncu_summary.py $R.ncu-rep > $O/sum_${1}_${2}.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/ncu_lines.py /dev/stdin 60 > $O/lines_${1}_${2}.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
for w in C5-cycle C5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'^k_' --csv --log-file $O/l_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e > $O/l_$w.log 2>&1; echo "list $w rc=$?"
python tools/ncu_summary.py --launches $O/l_$w.csv > $O/l_$w.txt 2>&1
done
