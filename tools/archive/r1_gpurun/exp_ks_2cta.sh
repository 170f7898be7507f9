#!/bin/bash
# ks_ntt_kernel at N = 2048 as two 512-thread CTAs per SM (one prime each, 8-column digit tiles;
# -DKS_EXP_2CTA, build C2) vs the final kernel (one 1024-thread CTA, both primes).
cd "$(dirname "$0")/../.."
for i in 1 2 3; do
for T in 256 1024; do
echo "== base T=$T"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py $T 2>&1 | grep "pack_ntt"
echo "== C2 T=$T"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_C2.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py $T 2>&1 | grep "pack_ntt\|ident"
done; done
