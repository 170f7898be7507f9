#!/bin/bash
# q_proj_packed at T = 2048: stage 1 on tcgen05 (default) vs the NTT-domain digits contraction.
mkdir -p gpurun_out
for c in tc ntt tc ntt; do
timeout 900 python bench.py --workload q_proj_packed --contraction $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/s1_$c.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/s1_$c.jsonl').read().strip().splitlines()[-1])
print('$c', d['value'], d['ms_per_step'], d.get('breakdown_ms'), d['clocks'].get('sm_mhz'))"
done
