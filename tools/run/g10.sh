set -x
timeout 1200 python -m pytest tests/test_gpu_gather.py tests/test_gpu_torchrun.py tests/test_gpu_p2p.py -q -x --durations=10 > gpurun_out/r2_g10_tests.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/r2_g10_tests.log
