set -x
timeout 1500 python -m pytest tests/test_gpu_pack_ntt.py tests/test_gpu_pack.py tests/test_gpu_wire.py tests/test_gpu_parity.py -q -x --durations=10 > gpurun_out/r2_g3_tests.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/r2_g3_tests.log
