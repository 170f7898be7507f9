set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_llama_linears.py tests/test_gpu_freivalds.py tests/test_gpu_pack.py -q -x > gpurun_out/r2_g4_tests.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r2_g4_tests.log
for T in 2040 2048 2091 16 60; do timeout 300 python tools/probe.py --T $T --reps 5; done
timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 5
