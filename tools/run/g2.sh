set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_gather.py tests/test_gpu_torchrun.py -q -x --durations=10 > gpurun_out/r2_g2_tests.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/r2_g2_tests.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_stack_s1.jsonl 2> gpurun_out/r2_bench_stack_s1.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/r2_bench_stack_s1.jsonl; tail -20 gpurun_out/r2_bench_stack_s1.err
