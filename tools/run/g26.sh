set -x
timeout 600 python bench.py --workload q_proj --steps 3 --warmup 3 > gpurun_out/r2_bench_q_proj.jsonl 2>gpurun_out/r2_bench_q_proj.err; echo "q rc=$?"; tail -c 500 gpurun_out/r2_bench_q_proj.jsonl
timeout 600 python bench.py --workload ffn --steps 3 --warmup 3 --no-e2e > gpurun_out/r2_bench_ffn.jsonl 2>&1; echo "ffn rc=$?"; tail -c 300 gpurun_out/r2_bench_ffn.jsonl
timeout 600 python bench.py --workload stack_packed --steps 3 --warmup 3 > gpurun_out/r2_bench_stack_packed.jsonl 2>&1; echo "sp rc=$?"; tail -c 300 gpurun_out/r2_bench_stack_packed.jsonl
timeout 600 python bench.py --workload q_proj_packed --steps 3 --warmup 3 > gpurun_out/r2_bench_q_proj_packed.jsonl 2>&1; echo "qp rc=$?"; tail -c 300 gpurun_out/r2_bench_q_proj_packed.jsonl
