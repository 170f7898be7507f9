#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack_ntt.py -x -q 2>&1 | tail -3
PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 256 2>&1 | tail -4
PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 16 2>&1 | tail -4
