for d in 0 1 2; do PHE_DEBUG_EPI=$d timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('dbg=$d', d['breakdown_ms']['mask_gemm'], d['clocks']['sm_mhz'], d['roofline']['frac'])"; done
python tools/probe.py --d_out 2048 --d_in 2048 --reps 10
python tools/probe.py --d_out 512 --d_in 8192 --reps 10
python tools/probe.py --d_out 2048 --d_in 8192 --reps 5
python tools/probe.py --d_out 8192 --d_in 2048 --T 512 --reps 10
python tools/probe.py --d_out 2048 --d_in 512 --transpose --reps 10
