echo "== base"; PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt"
for v in S0 S1 S2; do echo "== $v"; PHE_LIB=$PWD/paper_2505_07329_b200/libphe_$v.so PYTHONPATH=. timeout 300 python tools/probe_pack_ntt.py 256 2>&1 | grep "pack_ntt\|ident"; done
