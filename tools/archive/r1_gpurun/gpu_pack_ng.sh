#!/bin/bash
PHE_PACK_HINTS=1 timeout 600 python -m pytest tests/test_gpu_pack.py -x -q 2>&1 | tail -1
for cfg in "21 0" "21 1" "41 1" "82 1"; do
  set -- $cfg
  echo "NG=$1 HINTS=$2"; PHE_PACK_NG=$1 PHE_PACK_HINTS=$2 timeout 900 python bench.py --workload q_proj_packed --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['breakdown_ms'], d['clocks']['sm_mhz'])"
done
for cfg in "21 1" "41 1"; do set -- $cfg
PHE_PACK_NG=$1 PHE_PACK_HINTS=$2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:pack_gemm -c 1 python tools/ncu_pack.py 102 2>&1 | grep -E "dram__bytes_read|duration|per_second"
done
