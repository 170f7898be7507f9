set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wire.py tests/test_gpu_freivalds.py -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
