M=gpu__time_duration.sum,sm__cycles_elapsed.avg
for d in 0 1 2; do
PHE_DEBUG_EPI=$d ncu --metrics $M --clock-control none -k regex:limb_gemm_2sm -c 2 --csv python tools/probe.py --reps 1 2>/dev/null | grep -E "limb_gemm_2sm" | tail -2 | awk -F'","' -v d=$d '{print "dbg="d, $(NF-2), $NF}'
done
PHE_DEBUG_EPI=4 python tools/probe.py --reps 2 2>&1 | tail -3
PHE_DEBUG_EPI=4 python tools/probe.py --reps 2 --d_out 512 --d_in 8192 2>&1 | tail -2
