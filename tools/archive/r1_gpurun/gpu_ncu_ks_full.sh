#!/bin/bash
# ncu --set full of the ks_ntt_kernel launch in bench.py's q_proj_packed configuration (T = 2048)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ks_ntt_kernel -c 1 \
  -o gpurun_out/prof_ks_ntt_bench python bench.py --workload q_proj_packed --profile --steps 1 --warmup 0 \
  --no-e2e --no-cpu-baseline > gpurun_out/ncu_ks_bench.log 2>&1
python tools/ncu_summary_ntt.py gpurun_out/prof_ks_ntt_bench.ncu-rep gpurun_out/r1_ncu_ks_ntt_kernel_bench.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/r1_ncu_ks_ntt_kernel_bench.json'))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__grid_size','stall_pct']: print(k, d[k])"
