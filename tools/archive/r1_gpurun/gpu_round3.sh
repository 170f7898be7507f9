mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
python tools/bit_error_study.py --trials 65536 --out gpurun_out/r1_fig4_bit_errors.csv > /dev/null 2>&1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --target-processes all python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck.log 2>&1; tail -4 gpurun_out/sanitizer_memcheck.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck.log 2>&1; tail -3 gpurun_out/sanitizer_racecheck.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python __graft_entry__.py smoke > gpurun_out/sanitizer_synccheck.log 2>&1; tail -3 gpurun_out/sanitizer_synccheck.log
