set -x
timeout 900 python -m pytest tests/test_gpu_example.py -q -x 2>&1 | tail -3
timeout 300 python tools/example_protocol.py --tokens 16
timeout 300 python tools/example_protocol.py --tokens 16 --packed
