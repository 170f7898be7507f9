echo "== base"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
echo "== zero-add"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_Z.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt\|ident"
echo "== base"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
echo "== zero-add"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_Z.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
