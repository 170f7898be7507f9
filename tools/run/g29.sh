set -x
timeout 1200 python -m pytest tests/test_gpu_pack_ntt.py tests/test_gpu_llama_linears.py -q -x -k "ntt or packed" > gpurun_out/r2_g29_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2_g29_tests.log
bash tools/build_variant.sh smem -DKS_LANE_XCHG=0 2>&1 | grep -i error
for v in prod smem prod smem; do
if [ $v = smem ]; then export PHE_LIB=paper_2505_07329_b200/libphe_smem.so; else unset PHE_LIB; fi
PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 2048 2048 | grep pack_ntt | sed "s/^/$v /"
done
