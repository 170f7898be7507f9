set -x
for W in 0 1; do PHE_KS_W64=$W PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 2048 2048; done
