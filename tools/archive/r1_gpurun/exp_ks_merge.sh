#!/bin/bash
# Training step (stack_packed, T = 16): ks_ntt with one prime per CTA (default at small grids) vs
# both primes per CTA (-DKS_EXP_MERGE_ALWAYS, build MA; swapped in on the box copy only).
cd "$(dirname "$0")/../.."
for i in 1 2; do
timeout 900 python bench.py --workload stack_packed --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', d['ms_per_step'])"
cp paper_2505_07329_b200/libphe.so /tmp/libphe_base.so; cp paper_2505_07329_b200/libphe_MA.so paper_2505_07329_b200/libphe.so
timeout 900 python bench.py --workload stack_packed --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('MA', d['ms_per_step'])"
cp /tmp/libphe_base.so paper_2505_07329_b200/libphe.so
done
