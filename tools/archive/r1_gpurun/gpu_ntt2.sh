#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ntt.py -x -q -k "8192 or crt or transpose or identical or sharding" 2>&1 | tail -5
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_mask_kernel -s 1 -c 1 -o gpurun_out/ncu_ntt_v1 python tools/ncu_ntt.py 2>&1 | tail -3
