set -x
bash tools/build_variant.sh eg3 -DPHE_EPI_GROUPS=3 2>&1 | grep -i error
for v in prod eg3 prod eg3; do
if [ $v = eg3 ]; then export PHE_LIB=paper_2505_07329_b200/libphe_eg3.so; else unset PHE_LIB; fi
timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 10 | sed "s/^/$v /"
timeout 300 python tools/probe.py --T 2048 --reps 30 | sed "s/^/$v /"
timeout 300 python tools/probe.py --d_out 768 --d_in 768 --T 2048 --reps 10 | sed "s/^/$v /"
timeout 300 python tools/probe.py --d_out 16384 --d_in 2048 --T 255 --reps 30 | sed "s/^/$v /"
done
