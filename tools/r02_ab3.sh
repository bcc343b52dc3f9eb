#!/bin/bash
# C4/C5 scan timing of three builds in one call: round-1 final (abtest/r1), 40d2f53 (abtest/pre), current
O=gpurun_out/ab3; mkdir -p $O
for rep in 1 2; do
  for v in r1 pre cur; do
    for w in C4 C5; do
      if [ $v = cur ]; then python tools/scan_bench.py --workload $w --iters 5 > $O/${v}_${w}_$rep.json 2>&1
      else python abtest/$v/tools/scan_bench.py --workload $w --iters 5 > $O/${v}_${w}_$rep.json 2>&1; fi
    done
  done
done
