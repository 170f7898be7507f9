#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_wire.py -x -q 2>&1 | grep -E "FAILED|passed|failed|Error" | head -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench_q_proj_final.jsonl 2> gpurun_out/bench_final.err
python3 -c "
import json; d=json.loads(open('gpurun_out/r1_bench_q_proj_final.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']); print(json.dumps(d['e2e']))"
tail -2 gpurun_out/bench_final.err
