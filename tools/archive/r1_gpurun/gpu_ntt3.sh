#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_ntt.py -x -q -k "not full_size" 2>&1 | tail -2
PHE_NTT_SPLIT=0 timeout 300 python -m pytest tests/test_gpu_ntt.py -x -q -k "not full_size" 2>&1 | tail -2
for v in 0 1; do
  echo "SPLIT=$v"; PHE_NTT_SPLIT=$v timeout 300 python tools/probe_ntt.py --reps 3 --dense 0 --shapes 2048x2048x2048,2048x8192x512 2>&1 | tail -2
done
