set -x
timeout 900 python -m pytest tests/test_gpu_fig4.py -q -x 2>&1 | tail -5
timeout 1200 python tools/bit_error_study.py --trials 65536 --sigma 0 8 24 --out gpurun_out/r2_fig4_bit_errors.csv
