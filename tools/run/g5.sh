set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_llama_linears.py tests/test_gpu_freivalds.py tests/test_gpu_pack.py tests/test_gpu_pack_ntt.py tests/test_gpu_p2p.py -q -x > gpurun_out/r2_g5_tests.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r2_g5_tests.log
timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 5
timeout 300 python tools/probe.py --d_out 768 --d_in 768 --T 2048 --reps 5
timeout 300 python tools/probe.py --T 2048 --reps 5
