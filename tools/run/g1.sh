set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
nproc
timeout 1500 python -m pytest tests/test_gpu_freivalds.py tests/test_gpu_parity.py tests/test_gpu_ntt.py -q -x --durations=15 2>&1 | tail -30
