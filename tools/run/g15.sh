set -x
timeout 1200 python -m pytest tests/test_gpu_torchrun.py tests/test_gpu_gather.py -q -x > gpurun_out/r2_g15_tests.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r2_g15_tests.log
