#!/bin/bash
# Session 3 re-entry check: full GPU suite, smoke, default line, packed line on HEAD.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final3_tests.log 2>&1; tail -3 gpurun_out/final3_tests.log
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final3_q_proj.jsonl 2> gpurun_out/final3.err
timeout 1200 python bench.py --workload q_proj_packed --no-cpu-baseline > gpurun_out/final3_q_proj_packed.jsonl 2>> gpurun_out/final3.err
for f in final3_q_proj final3_q_proj_packed; do
python -c "
import json; d=json.loads(open('gpurun_out/$f.jsonl').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
done
tail -2 gpurun_out/final3.err
