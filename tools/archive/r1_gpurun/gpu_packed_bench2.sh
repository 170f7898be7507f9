#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack_ntt.py -x -q 2>&1 | tail -1
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 16 2>&1 | grep "pack_ntt"
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 1 2>&1 | grep "pack"
timeout 1200 python bench.py --workload stack_packed --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_stack_packed_ntt_ksntt.jsonl 2> gpurun_out/pk.err; tail -1 gpurun_out/r1_bench_stack_packed_ntt_ksntt.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['breakdown_ms'])"
