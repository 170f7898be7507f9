#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_wire.py tests/test_gpu_pack.py -x -q 2>&1 | grep -E "FAILED|passed|failed|Error" | head -3
timeout 900 python tools/side_bw.py --reps 5 2>&1 | grep wire
