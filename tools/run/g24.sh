set -x
timeout 1200 python bench.py --bwd fused --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_stack_fusedbwd.jsonl 2> gpurun_out/r2_bench_stack_fusedbwd.err
echo "rc=$?"; tail -c 1200 gpurun_out/r2_bench_stack_fusedbwd.jsonl
