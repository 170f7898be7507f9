set -x
bash tools/build_variant.sh exp -DPHE_KERNEL_EXPERIMENTS=1 2>&1 | grep -i error
for D in 0 1; do
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_EPI_DIRECT=$D timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 5
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_EPI_DIRECT=$D timeout 300 python tools/probe.py --T 2048 --reps 5
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_EPI_DIRECT=$D timeout 300 python tools/probe.py --d_out 768 --d_in 768 --T 2048 --reps 5
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_EPI_DIRECT=$D timeout 300 python tools/probe.py --d_out 8192 --d_in 2048 --T 510 --reps 5
done
