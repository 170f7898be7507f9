#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q -k "digits" 2>&1 | grep -E "FAILED|passed|failed|Error" | head -3
timeout 900 python -m pytest tests/test_gpu_pack.py -x -q 2>&1 | tail -1
timeout 1200 python bench.py --workload stack_packed --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_ntt.jsonl 2>/dev/null
timeout 900 python bench.py --workload q_proj_packed --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_packed_ntt.jsonl 2>/dev/null
for f in gpurun_out/r1_bench_stack_packed_ntt.jsonl gpurun_out/r1_bench_q_proj_packed_ntt.jsonl; do python3 -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['breakdown_ms'], (d.get('e2e') or {}).get('value'))"; done
