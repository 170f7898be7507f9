set -x
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_stack_s2.jsonl 2> gpurun_out/r2_bench_stack_s2.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/r2_bench_stack_s2.jsonl
# launch list of one step of a 1-layer stack (after 3 warm-up steps: 3 x 99 x ~3 launches)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/r2_launches_stack1.csv python bench.py --layers 1 --steps 1 --warmup 3 --profile --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu list rc=$?"
# one gate_up chunk mask launch (255 tokens, 16384 rows) of the stack, full set
timeout 900 ncu --set full --clock-control none --import-source on -k regex:limb_gemm_2sm -s 2 -c 1 -o gpurun_out/r2_ncu_stack_gateup python bench.py --layers 1 --steps 1 --warmup 3 --profile --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu full rc=$?"; ls -la gpurun_out/
