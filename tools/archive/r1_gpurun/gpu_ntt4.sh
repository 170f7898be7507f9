#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_ntt.py -x -q -k "not full_size" 2>&1 | grep -E "FAILED|passed|failed" | head -3
timeout 300 python tools/probe_ntt.py --reps 3 --dense 0 --shapes 2048x2048x2048,2048x8192x512 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_mask_kernel -s 1 -c 1 -o gpurun_out/ncu_ntt_A2 python tools/ncu_ntt.py 2>&1 | tail -1
