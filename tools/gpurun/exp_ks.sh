timeout 1200 python -m pytest tests/test_gpu_pack_ntt.py tests/test_gpu_pack.py -q 2>&1 | tail -1
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
timeout 1200 python bench.py --workload q_proj_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_q_proj_packed_ksntt.jsonl 2> gpurun_out/pk.err
timeout 1200 python bench.py --workload stack_packed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_default.jsonl 2>> gpurun_out/pk.err
for f in r1_bench_q_proj_packed_ksntt r1_bench_stack_packed_default; do python -c "
import json; d=json.loads(open('gpurun_out/$f.jsonl').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d['breakdown_ms'], d['clocks']['sm_mhz'])"; done
