#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q 2>&1 | grep -E "FAILED|passed|failed|Error" | head -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python tools/sweep.py --tokens 2048 2>&1 | grep '"ntt"' | cut -c1-200
