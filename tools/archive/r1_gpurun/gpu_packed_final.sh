#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --workload q_proj_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_packed_ksntt.jsonl 2> gpurun_out/pk.err
timeout 1200 python bench.py --workload stack_packed --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_ntt_ksntt.jsonl 2>> gpurun_out/pk.err
for f in gpurun_out/r1_bench_q_proj_packed_ksntt.jsonl gpurun_out/r1_bench_stack_packed_ntt_ksntt.jsonl; do
python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d['breakdown_ms'], d['clocks']['sm_mhz'])"
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ks_ntt_kernel -c 1 \
  -o gpurun_out/prof_ks_ntt_bench python bench.py --workload q_proj_packed --profile --steps 1 --warmup 0 \
  --no-e2e --no-cpu-baseline > gpurun_out/ncu_ks_bench.log 2>&1
python tools/ncu_summary_ntt.py gpurun_out/prof_ks_ntt_bench.ncu-rep gpurun_out/r1_ncu_ks_ntt_kernel_bench.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/r1_ncu_ks_ntt_kernel_bench.json'))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__grid_size','stall_pct']: print(k, d[k])"
