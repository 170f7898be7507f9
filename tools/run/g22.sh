set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_freivalds.py tests/test_gpu_llama_linears.py tests/test_gpu_wire.py tests/test_gpu_pack.py -q -x > gpurun_out/r2_g22_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r2_g22_tests.log
bash tools/build_variant.sh exp -DPHE_KERNEL_EXPERIMENTS=1 2>&1 | grep -i error
for e in 0 1 0 1; do
if [ $e = 1 ]; then export PHE_NACC2=1; else unset PHE_NACC2; fi
PHE_LIB=paper_2505_07329_b200/libphe_exp.so timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 20 | sed "s/^/nacc2=$e /"
done
unset PHE_NACC2
timeout 300 python tools/probe.py --d_out 512 --d_in 2048 --transpose --T 2048 --reps 20 | sed "s/^/prod /"
timeout 300 python tools/probe.py --d_out 768 --d_in 768 --T 2048 --reps 20 | sed "s/^/prod /"
