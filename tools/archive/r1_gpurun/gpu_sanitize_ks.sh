#!/bin/bash
# compute-sanitizer on the NTT KeySwitch parity tests (small rings + the Table 1 ring)
mkdir -p gpurun_out
K="test_pack_ntt_bit_exact_vs_oracle or test_pack_ntt_crt_range or identical_to_tensor_core and 2048-2048"
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --target-processes all \
    python -m pytest tests/test_gpu_pack_ntt.py -x -q -k "$K" > gpurun_out/r1_sanitizer_${tool}_ks_ntt.log 2>&1
  echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/r1_sanitizer_${tool}_ks_ntt.log | tail -4
done
