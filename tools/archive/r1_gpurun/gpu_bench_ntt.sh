#!/bin/bash
# NEXT #4 measurement: q_proj (configs[1]) through the NTT path, FFN (configs[2]) ntt/hybrid,
# and the tc default for comparison in the same session.
mkdir -p gpurun_out
timeout 900 python bench.py --contraction ntt --steps 5 --warmup 3 > gpurun_out/r1_bench_q_proj_ntt.jsonl 2> gpurun_out/bench_ntt.err; tail -1 gpurun_out/r1_bench_q_proj_ntt.jsonl | cut -c1-400
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/r1_bench_q_proj_tc_same_box.jsonl 2>>gpurun_out/bench_ntt.err; tail -1 gpurun_out/r1_bench_q_proj_tc_same_box.jsonl | cut -c1-300
timeout 1200 python bench.py --workload ffn --contraction hybrid --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_ffn_hybrid.jsonl 2>>gpurun_out/bench_ntt.err; tail -1 gpurun_out/r1_bench_ffn_hybrid.jsonl | cut -c1-300
timeout 1200 python bench.py --workload ffn --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_ffn_tc.jsonl 2>>gpurun_out/bench_ntt.err; tail -1 gpurun_out/r1_bench_ffn_tc.jsonl | cut -c1-300
tail -5 gpurun_out/bench_ntt.err
