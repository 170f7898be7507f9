set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pack.py tests/test_gpu_wire.py tests/test_gpu_p2p.py tests/test_gpu_gather.py -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
