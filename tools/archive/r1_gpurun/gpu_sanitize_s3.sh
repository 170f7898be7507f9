#!/bin/bash
# compute-sanitizer on this session's new device code: the shared-memory-staged wire kernels
# (test_gpu_wire.py) and the all-NTT packed primitive + its wire host pipeline (nttw cases).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --target-processes all \
    python -m pytest tests/test_gpu_wire.py tests/test_gpu_pack_ntt.py -x -q -k "wire or empty_and_errors" \
    > gpurun_out/r1_sanitizer_${tool}_s3.log 2>&1
  echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/r1_sanitizer_${tool}_s3.log | tail -4
done
