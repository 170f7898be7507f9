#!/bin/bash
for c in 0 1 2 3; do
  PHE_NTT_CFG=$c timeout 300 python -m pytest tests/test_gpu_ntt.py -x -q -k "not full_size" 2>&1 | grep -E "FAILED|passed|failed" | head -2
  echo "CFG=$c"; PHE_NTT_CFG=$c timeout 300 python tools/probe_ntt.py --reps 3 --dense 0 --shapes 2048x2048x2048,2048x8192x512 2>&1 | tail -2
done
