#!/bin/bash
# ks_ntt digit-tile cp.async with the L2::128B prefetch qualifier: parity, DRAM bytes of the bench
# launch, and the packed default line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pack_ntt.py -q -x 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ks_ntt_kernel -c 1 --csv \
  python bench.py --workload q_proj_packed --profile --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
for i in 1 2; do
timeout 900 python bench.py --workload q_proj_packed --no-cpu-baseline --no-e2e --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('breakdown_ms'), d['clocks']['sm_mhz'])"
done
