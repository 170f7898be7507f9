set -x
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --launch-timeout 0 python -m pytest tests/test_gpu_parity.py -q -x -k "paper_params or partial_block or empty_and_single or row_sharding" > gpurun_out/r2_sanitizer_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -4 gpurun_out/r2_sanitizer_memcheck.log
timeout 1500 compute-sanitizer --tool synccheck --launch-timeout 0 python -m pytest tests/test_gpu_parity.py -q -x -k "paper_params or partial_block" > gpurun_out/r2_sanitizer_synccheck.log 2>&1
echo "synccheck rc=$?"; tail -4 gpurun_out/r2_sanitizer_synccheck.log
timeout 1500 compute-sanitizer --tool racecheck --launch-timeout 0 python -m pytest tests/test_gpu_parity.py -q -x -k "partial_block" > gpurun_out/r2_sanitizer_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -6 gpurun_out/r2_sanitizer_racecheck.log
