#!/bin/bash
# ncu --set full of one ks_ntt_kernel launch (stage 2 of the packed primitive, NTT domain)
mkdir -p gpurun_out
PYTHONPATH=. timeout 900 ncu --set full --clock-control none --import-source on -k regex:ks_ntt_kernel -s 1 -c 1 \
  -o gpurun_out/prof_ks_ntt python tools/probe_pack_ntt.py 32 > gpurun_out/ncu_ks.log 2>&1
tail -3 gpurun_out/ncu_ks.log
python tools/ncu_summary_ntt.py gpurun_out/prof_ks_ntt.ncu-rep gpurun_out/ncu_ks_ntt.json > /dev/null 2>&1
ls -la gpurun_out/prof_ks_ntt.ncu-rep
