set -x
timeout 900 python -m pytest tests/test_gpu_wire.py -q -x 2>&1 | tail -3
