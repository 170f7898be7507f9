#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack_ntt.py tests/test_gpu_pack.py -x -q 2>&1 | tail -2
timeout 1200 python bench.py --workload q_proj_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_packed_ksntt.jsonl 2> gpurun_out/pk.err; tail -1 gpurun_out/r1_bench_q_proj_packed_ksntt.jsonl
timeout 1200 python bench.py --workload stack_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_ksntt.jsonl 2>> gpurun_out/pk.err; tail -1 gpurun_out/r1_bench_stack_packed_ksntt.jsonl
timeout 1200 python bench.py --workload stack_packed --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_ntt_ksntt.jsonl 2>> gpurun_out/pk.err; tail -1 gpurun_out/r1_bench_stack_packed_ntt_ksntt.jsonl
tail -3 gpurun_out/pk.err
