#!/bin/bash
# Both packed stages in the NTT domain: parity (library + wire host pipeline), the two-rank bench
# test, and the default q_proj_packed line (e2e through phe_server_wire_host_nttw, checked against
# the device step's outputs).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack_ntt.py tests/test_gpu_torchrun.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --workload q_proj_packed --no-cpu-baseline > gpurun_out/nttw_packed.jsonl 2> gpurun_out/nttw.err
python -c "
import json; d=json.loads(open('gpurun_out/nttw_packed.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['config'].get('contraction'), d.get('breakdown_ms'), d['e2e'], d['roofline']['frac'], d['clocks'])"
tail -3 gpurun_out/nttw.err
