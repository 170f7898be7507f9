#!/bin/bash
# ks_ntt_kernel floor: forward NTT and pointwise stage both dropped (timing-only build FL).
cd "$(dirname "$0")/../.."
for i in 1 2; do
echo "== base"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
echo "== FL"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_FL.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
done
