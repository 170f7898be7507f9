#!/bin/bash
# Final measurement pass (round 1): every bench line in profiles/ regenerated with the final build.
mkdir -p gpurun_out
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_torchrun1.jsonl 2> gpurun_out/final.err
timeout 2400 python bench.py --workload stack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack.jsonl 2>> gpurun_out/final.err
timeout 1500 python bench.py --workload ffn --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_ffn_tc.jsonl 2>> gpurun_out/final.err
timeout 1200 python bench.py --workload q_proj_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_packed.jsonl 2>> gpurun_out/final.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1_bench_reference.jsonl 2>> gpurun_out/final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r1_launches_q_proj.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>> gpurun_out/final.err
set +x
for f in gpurun_out/r1_bench_q_proj_torchrun1.jsonl gpurun_out/r1_bench_stack.jsonl gpurun_out/r1_bench_ffn_tc.jsonl gpurun_out/r1_bench_q_proj_packed.jsonl gpurun_out/r1_bench_reference.jsonl; do
python3 -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f'.split('/')[-1], d.get('value'), d.get('ms_per_step'), r.get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'))"
done
tail -3 gpurun_out/final.err
