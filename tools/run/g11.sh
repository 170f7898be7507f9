set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:limb_gemm_2sm -s 2 -c 1 -o gpurun_out/r2_ncu_kT python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 1 > /dev/null 2>&1
echo "ncu rc=$?"
