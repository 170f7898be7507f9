timeout 900 python -m pytest tests/test_gpu_pack_ntt.py -x -q 2>&1 | tail -1
echo "== shoup"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt\|ident"
PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 16 2>&1 | grep "pack_ntt"
echo "== mont"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_M.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
