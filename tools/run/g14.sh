set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2_gpu_tests_s2.log 2>&1
echo "pytest rc=$?"; tail -22 gpurun_out/r2_gpu_tests_s2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_stack_s3.jsonl 2> gpurun_out/r2_bench_stack_s3.err
echo "bench rc=$?"; tail -c 600 gpurun_out/r2_bench_stack_s3.jsonl
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference_s3.jsonl 2>&1
echo "ref rc=$?"; tail -c 400 gpurun_out/r2_bench_reference_s3.jsonl
