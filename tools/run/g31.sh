set -x
bash tools/build_variant.sh exp -DPHE_KERNEL_EXPERIMENTS=1 2>&1 | grep -i error
for d in 0 9 4; do PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_DEBUG_EPI=$d timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 10 2>&1 | sed "s/^/kT dbg$d /"; done
for d in 9; do PHE_NO_JPAIR=1 PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_DEBUG_EPI=$d timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 10 2>&1 | sed "s/^/kT nojpair dbg$d /"; done
PHE_LIB=paper_2505_07329_b200/libphe_exp.so PHE_DEBUG_EPI=4 timeout 300 python tools/probe.py --d_out 2048 --d_in 2048 --transpose --T 2048 --reps 10 2>&1 | sed "s/^/qT dbg4 /"
