set -x
timeout 1500 compute-sanitizer --tool memcheck --launch-timeout 0 python -m pytest tests/test_gpu_wire.py -q -x > gpurun_out/r2_sanitizer_memcheck_wire.log 2>&1
echo "memcheck rc=$?"; tail -4 gpurun_out/r2_sanitizer_memcheck_wire.log
timeout 1500 compute-sanitizer --tool synccheck --launch-timeout 0 python -m pytest tests/test_gpu_wire.py -q -x -k "matmul_clear_wire" > gpurun_out/r2_sanitizer_synccheck_wire.log 2>&1
echo "synccheck rc=$?"; tail -3 gpurun_out/r2_sanitizer_synccheck_wire.log
timeout 1500 compute-sanitizer --tool racecheck --launch-timeout 0 python -m pytest tests/test_gpu_wire.py -q -x -k "equals_serialized and 300" > gpurun_out/r2_sanitizer_racecheck_wire.log 2>&1
echo "racecheck rc=$?"; grep -c "Race reported" gpurun_out/r2_sanitizer_racecheck_wire.log; grep "Race reported" -A2 gpurun_out/r2_sanitizer_racecheck_wire.log | grep "limb_gemm.cu" | sed 's/.*limb_gemm.cu/limb_gemm.cu/' | sort | uniq -c
