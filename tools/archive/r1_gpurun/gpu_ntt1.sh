#!/bin/bash
# NEXT #4 first GPU pass: NTT parity tests, then timing probe vs the tensor-core path.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q 2>&1 | tail -25 > gpurun_out/ntt_tests.log
cat gpurun_out/ntt_tests.log
timeout 600 python tools/probe_ntt.py --reps 3 2>&1 | tail -10 | tee gpurun_out/ntt_probe.log
