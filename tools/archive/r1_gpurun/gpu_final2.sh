#!/bin/bash
# Final measurement pass (session 2): full GPU suite, smoke, default line, reference arm, packed lines.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final2_tests.log 2>&1; tail -2 gpurun_out/final2_tests.log
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r1_bench_q_proj_final.jsonl 2> gpurun_out/final2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1_bench_reference.jsonl 2>> gpurun_out/final2.err
timeout 1200 python bench.py --workload stack_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_default.jsonl 2>> gpurun_out/final2.err
for f in r1_bench_q_proj_final r1_bench_reference r1_bench_stack_packed_default; do
python -c "
import json; d=json.loads(open('gpurun_out/$f.jsonl').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
done
tail -2 gpurun_out/final2.err
