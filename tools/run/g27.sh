set -x
bash tools/build_variant.sh exp -DPHE_KERNEL_EXPERIMENTS=1 2>&1 | grep -i error
for S in 1 4 8 16 1; do PHE_KS_SPLITS=$S PHE_LIB=paper_2505_07329_b200/libphe_exp.so PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 2048 2048 | grep pack_ntt | sed "s/^/S=$S /"; done
for S in 1 8; do PHE_KS_SPLITS=$S PHE_LIB=paper_2505_07329_b200/libphe_exp.so PYTHONPATH=. timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:ks_ntt_kernel -c 1 python tools/probe_pack_ntt.py 2048 2048 2>/dev/null | grep -E "dram__bytes|gpu__time" | sed "s/^/S=$S /"; done
