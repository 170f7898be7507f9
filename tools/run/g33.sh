set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r2_gpu_tests_final.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/r2_gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_stack_final.jsonl 2> gpurun_out/r2_bench_stack_final.err
echo "bench rc=$?"; tail -c 700 gpurun_out/r2_bench_stack_final.jsonl
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference_final.jsonl 2>&1
echo "ref rc=$?"; tail -c 300 gpurun_out/r2_bench_reference_final.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/r2_launches_stack1_final.csv python bench.py --layers 1 --steps 1 --warmup 3 --profile --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu rc=$?"
