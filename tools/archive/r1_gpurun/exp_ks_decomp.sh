#!/bin/bash
# Time decomposition of ks_ntt_kernel (T = 256 probe): K_hat loads made L1-hot, pointwise stage
# dropped, forward NTT dropped (timing-only builds, outputs wrong by construction).
cd "$(dirname "$0")/../.."
if [ "$1" = build ]; then for v in "KH -DKS_EXP_KHAT_FIXED" "NP -DKS_EXP_NO_POINTWISE" "NN -DKS_EXP_NO_NTT"; do
  set -- $v; bash tools/gpurun/build_variant.sh $1 $2 &
done; wait; fi
for i in 1 2; do
echo "== base"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
for n in KH NP NN; do echo "== $n"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_$n.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt\|ident"; done
done
