#!/bin/bash
O=gpurun_out/p40; mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu_extra.py -m gpu -q -x -k "row_shard" > $O/t.log 2>&1; echo "t rc=$?"; tail -15 $O/t.log
