#!/bin/bash
# Shared-memory-staged wire kernels: parity suites that cover the wire format, then the side-kernel
# bandwidth report (+ ncu DRAM bytes) into gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wire.py tests/test_gpu_pack_ntt.py tests/test_gpu_pack.py -q -x 2>&1 | tail -3
bash tools/gpurun/gpu_side_bw.sh
