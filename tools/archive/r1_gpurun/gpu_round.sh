# One gpurun call: full-size parity test, ncu launch list + full capture of the mask kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and slow" -x -q 2>&1 | tail -3 > gpurun_out/slow_test.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --profile --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:limb_gemm_2sm -c 1 -o gpurun_out/prof_mask_r1 python bench.py --profile --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_r1.log 2>&1
cat gpurun_out/slow_test.log
