#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --contraction ntt --steps 5 --warmup 3 > gpurun_out/r1_bench_q_proj_ntt.jsonl 2> gpurun_out/bench_ntt.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/r1_bench_q_proj_tc_same_box.jsonl 2>>gpurun_out/bench_ntt.err
timeout 1500 python bench.py --workload ffn --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_ffn_ntt.jsonl 2>>gpurun_out/bench_ntt.err
timeout 1500 python bench.py --workload ffn --contraction hybrid --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_ffn_hybrid.jsonl 2>>gpurun_out/bench_ntt.err
timeout 1500 python bench.py --workload ffn --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_ffn_tc.jsonl 2>>gpurun_out/bench_ntt.err
timeout 2400 python bench.py --workload stack --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_ntt.jsonl 2>>gpurun_out/bench_ntt.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_mask_kernel -s 1 -c 1 -o gpurun_out/ncu_ntt_final python tools/ncu_ntt.py > /dev/null 2>&1
for f in gpurun_out/r1_bench_*ntt*.jsonl gpurun_out/r1_bench_q_proj_tc_same_box.jsonl gpurun_out/r1_bench_ffn_*.jsonl; do echo "$f $(tail -1 $f | cut -c1-200)"; done
tail -3 gpurun_out/bench_ntt.err
