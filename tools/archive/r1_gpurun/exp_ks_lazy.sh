#!/bin/bash
# ks_ntt_kernel: lazy accumulation (reduce every 7 products, -DKS_EXP_LAZY_ACC, build LA) vs base.
cd "$(dirname "$0")/../.."
for i in 1 2 3; do
echo "== base"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
echo "== LA"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_LA.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt\|ident"
done
