#!/bin/bash
PHE_NTT_NG4=1 timeout 600 python -m pytest tests/test_gpu_ntt.py -x -q 2>&1 | grep -E "FAILED|passed|failed|Error" | head -3
for v in 0 1; do echo "NG4=$v"; PHE_NTT_NG4=$v timeout 300 python tools/probe_ntt.py --reps 3 --dense 0 --shapes 2048x2048x2048 2>&1 | tail -1; done
for t in 16 32; do echo "NG4=1 TOK=$t"; PHE_NTT_TOK=$t PHE_NTT_NG4=1 timeout 300 python tools/probe_ntt.py --reps 3 --dense 0 --shapes 2048x2048x2048 2>&1 | tail -1; done
