#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_pack_ntt.py -x -q -k full_size --durations=3 2>&1 | tail -6
