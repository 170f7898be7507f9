#!/bin/bash
# Full GPU suite with the NTT KeySwitch, packed-workload launch list (ncu), q_proj_packed tc line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r4_tests.log 2>&1; tail -2 gpurun_out/r4_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r1_launches_q_proj_packed_ksntt.csv \
  python bench.py --workload q_proj_packed --tokens 510 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/r4.err
timeout 1200 python bench.py --workload q_proj_packed --pack tc --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_packed_tc_same_box.jsonl 2>> gpurun_out/r4.err
tail -1 gpurun_out/r1_bench_q_proj_packed_tc_same_box.jsonl | cut -c1-300
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r1_launches_q_proj_packed_ksntt.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
tot={}
for r in rows[1:]:
    k=r[ik].split('(')[0][:60]; tot[k]=tot.get(k,0)+float(r[iv].replace(',',''))
s=sum(tot.values())
for k,v in sorted(tot.items(), key=lambda kv:-kv[1])[:8]: print(f"{v/1e6:9.2f} ms {100*v/s:5.1f}%  {k}")
PY
