#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_ntt.py -x -q 2>&1 | grep -E "FAILED|passed|failed|Error" | head -5
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 300 python tools/probe_ntt.py --reps 3 --dense 0 --shapes 2048x2048x2048,2048x8192x2048,8192x2048x512 2>&1 | tail -3
