#!/bin/bash
# tensor-core modular GEMM: parity tests, then C5-cycle bench A/B (tcgen05 vs CUDA cores)
O=gpurun_out/p29; mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "cycle_gemm" > $O/t.log 2>&1; echo "t rc=$?"; tail -15 $O/t.log
timeout 300 python bench.py --workload C5-cycle --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_tc.log 2>&1; echo "tc rc=$?"
COMPASS_GEMM=cuda timeout 300 python bench.py --workload C5-cycle --steps 5 --warmup 3 --no-e2e --no-cpu > $O/b_cuda.log 2>&1; echo "cuda rc=$?"
for f in b_tc b_cuda; do grep '^{' $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['timing'], d['estimates'][:3] if 'estimates' in d else '')"; done
