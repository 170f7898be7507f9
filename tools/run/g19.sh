set -x
bash tools/build_variant.sh exp -DPHE_KERNEL_EXPERIMENTS=1 2>&1 | grep -i error
for d in 0 7 8 0 7 8; do PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_DEBUG_EPI=$d timeout 300 python tools/probe.py --T 2048 --reps 60 | sed "s/^/dbg$d /"; done
