M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for d in 0 1 2; do
PHE_DEBUG_EPI=$d ncu --metrics $M --clock-control none -k regex:limb_gemm_2sm -c 2 --csv python tools/probe.py --reps 1 2>/dev/null | grep -E "limb_gemm_2sm" | tail -4 | awk -F'","' -v d=$d '{print "dbg="d, $(NF-2), $NF}'
done
for shape in "--d_out 512 --d_in 8192" "--d_out 8192 --d_in 2048 --T 512"; do
ncu --metrics $M --clock-control none -k regex:limb_gemm_2sm -c 2 --csv python tools/probe.py $shape --reps 1 2>/dev/null | grep -E "limb_gemm_2sm" | tail -4 | awk -F'","' -v d="$shape" '{print d, $(NF-2), $NF}'
done
