#!/bin/bash
for cfg in "14 1" "16 1" "21 1" "28 1"; do
  set -- $cfg
  echo "NG=$1 HINTS=$2"; PHE_PACK_NG=$1 PHE_PACK_HINTS=$2 timeout 900 python bench.py --workload q_proj_packed --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['breakdown_ms']['pack_gemm_finalize'], d['clocks']['sm_mhz'])"
done
