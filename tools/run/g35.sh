set -x
timeout 1500 python -m pytest tests/test_gpu_freivalds.py -q -x -k "qkv_T or gate_up_T" --durations=4 2>&1 | tail -8
