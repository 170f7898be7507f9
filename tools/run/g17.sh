set -x
bash tools/build_variant.sh exp -DPHE_KERNEL_EXPERIMENTS=1 2>&1 | grep -i error
for rep in 1 2; do
for v in "0 0" "1 0" "0 1" "1 1"; do set -- $v
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_STORE_HINT=$1 PHE_LOAD_HINT=$2 timeout 300 python tools/probe.py --T 2048 --reps 60 | sed "s/^/S$1L$2 /"
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_STORE_HINT=$1 PHE_LOAD_HINT=$2 timeout 300 python tools/probe.py --d_out 16384 --d_in 2048 --T 255 --reps 40 | sed "s/^/S$1L$2 /"
done; done
