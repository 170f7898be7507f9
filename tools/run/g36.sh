set -x
timeout 2400 compute-sanitizer --tool memcheck --launch-timeout 0 python -m pytest tests/test_gpu_pack_ntt.py tests/test_gpu_pack.py tests/test_gpu_ntt.py -q -x -k "not full_size and not bench_config" > gpurun_out/r2_sanitizer_memcheck_hostpipes.log 2>&1
echo "memcheck rc=$?"; tail -5 gpurun_out/r2_sanitizer_memcheck_hostpipes.log
