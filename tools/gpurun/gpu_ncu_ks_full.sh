#!/bin/bash
# ncu --set full of the ks_ntt_kernel launch in bench.py's q_proj_packed configuration (T = 2048)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ks_ntt_kernel -c 1 \
  -o gpurun_out/prof_ks_ntt_bench python bench.py --workload q_proj_packed --profile --steps 1 --warmup 0 \
  --no-e2e --no-cpu-baseline > gpurun_out/ncu_ks_bench.log 2>&1
tail -2 gpurun_out/ncu_ks_bench.log
python tools/ncu_summary_ntt.py gpurun_out/prof_ks_ntt_bench.ncu-rep gpurun_out/r1_ncu_ks_ntt_kernel_bench.json | head -12
