#!/bin/bash
# Session-3 final pass: full GPU suite, smoke, default line, reference arm, training step, and the
# ncu launch list of the packed default (both stages in the NTT domain).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final4_tests.log 2>&1; tail -2 gpurun_out/final4_tests.log
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final4_q_proj.jsonl 2> gpurun_out/final4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final4_reference.jsonl 2>> gpurun_out/final4.err
timeout 1200 python bench.py --workload stack_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final4_stack_packed.jsonl 2>> gpurun_out/final4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r1_launches_q_proj_packed_nttw.csv \
  python bench.py --workload q_proj_packed --tokens 510 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>> gpurun_out/final4.err
for f in final4_q_proj final4_reference final4_stack_packed; do
python -c "
import json; d=json.loads(open('gpurun_out/$f.jsonl').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
done
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r1_launches_q_proj_packed_nttw.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
tot={}
for r in rows[1:]:
    k=r[ik].split('(')[0][:60]; tot[k]=tot.get(k,0)+float(r[iv].replace(',',''))
s=sum(tot.values())
for k,v in sorted(tot.items(), key=lambda kv:-kv[1])[:8]: print(f"{v/1e6:9.2f} ms {100*v/s:5.1f}%  {k}")
PY
tail -2 gpurun_out/final4.err
