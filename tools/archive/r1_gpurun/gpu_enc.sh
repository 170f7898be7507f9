#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q -k encrypt 2>&1 | grep -E "FAILED|passed|failed|Error" | head -3
timeout 600 python tools/side_bw.py --reps 5 2>&1 | grep -i encrypt | cut -c1-160
