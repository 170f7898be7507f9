#!/bin/bash
# NTT digits epilogue with quad-shuffled word stores: parity (digits == tensor-core digits, packed
# primitive per Llama shape) and the stage-1 kernel time in the packed bench configuration.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_llama_linears.py tests/test_gpu_pack_ntt.py -q -x 2>&1 | tail -2
for i in 1 2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ntt_mask_kernel -c 1 --csv \
  python bench.py --workload q_proj_packed --profile --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>/dev/null | grep gpu__time | awk -F'","' '{print "stage1 ms", $NF}'
done
timeout 900 python bench.py --workload q_proj_packed --no-cpu-baseline > gpurun_out/digw_packed.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/digw_packed.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d.get('breakdown_ms'), d['e2e']['value'], d['e2e']['output_equals_device_step'], d['clocks']['sm_mhz'])"
