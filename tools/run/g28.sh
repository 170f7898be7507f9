set -x
timeout 1500 python tools/table3.py > gpurun_out/r2_table3.log 2>&1; echo "rc=$?"; tail -12 gpurun_out/r2_table3.log
