timeout 900 python -m pytest tests/test_gpu_pack_ntt.py -x -q 2>&1 | tail -1
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 16 2>&1 | grep "pack_ntt"
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 2048 2>&1 | grep "pack_ntt\|ident"
