set -x
timeout 600 python bench.py --layers 2 --tokens 100 --steps 3 --warmup 3 > gpurun_out/r2_b_small.jsonl 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/r2_b_small.jsonl
timeout 600 python bench.py --layers 2 --tokens 300 --contraction hybrid --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b_hybrid.jsonl 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/r2_b_hybrid.jsonl
timeout 600 python bench.py --layers 1 --tokens 64 --contraction ntt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b_ntt.jsonl 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/r2_b_ntt.jsonl
timeout 600 python bench.py --layers 1 --tokens 40 --bwd fused --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b_fused.jsonl 2>&1; echo "rc=$?"; tail -c 300 gpurun_out/r2_b_fused.jsonl
