set -x
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r2_gpu_tests_s3.log 2>&1
echo "pytest rc=$?"; tail -10 gpurun_out/r2_gpu_tests_s3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
