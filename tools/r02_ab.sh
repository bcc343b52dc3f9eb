#!/bin/bash
# A/B of two library builds within one call: tools/r02_ab.sh OUT LIB_A LIB_B workload...
O=$1; A=$2; B=$3; shift 3
mkdir -p $O
for w in "$@"; do
  for rep in 1 2; do
    COMPASS_LIB=$A python tools/scan_bench.py --workload $w --iters 5 > $O/a_${w}_$rep.json 2>&1
    COMPASS_LIB=$B python tools/scan_bench.py --workload $w --iters 5 > $O/b_${w}_$rep.json 2>&1
  done
done
