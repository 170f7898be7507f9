M=gpu__time_duration.sum,sm__cycles_elapsed.avg
for d in 0 1 2 7 8; do
PHE_DEBUG_EPI=$d ncu --metrics $M --clock-control none -k regex:limb_gemm_2sm -c 2 --csv python tools/probe.py --reps 1 2>/dev/null | grep -E "limb_gemm_2sm" | tail -1 | awk -F'","' -v d=$d '{print "dbg="d, $(NF-2), $NF}'
done
