set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r2_gpu_tests.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/r2_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
