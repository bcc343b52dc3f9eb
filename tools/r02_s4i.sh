#!/bin/bash
# cross-GPU merge over peer memory (fused push): GPU tests, bench N=1 nccl vs peer, scan regressions
O=gpurun_out/s4i; mkdir -p $O
timeout 900 python -m pytest tests/test_peer_merge_gpu.py -m gpu -q -x > $O/t_peer.log 2>&1; echo "peer tests rc=$?"; tail -15 $O/t_peer.log
for m in nccl peer; do
  for w in C4 C5; do
    timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --merge $m > $O/b_${w}_$m.log 2>&1
    grep '^{' $O/b_${w}_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; print('$w $m', t['build_ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac'], d['gpu_launches'])"
  done
done
