#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/side_bw.py --reps 5 2>&1 | tail -12
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"modswitch|decrypt_kernel|encrypt_kernel|ct_prepare|wire_|ntt_masks" --csv --log-file gpurun_out/r1_side_kernels_ncu.csv python tools/side_bw.py --reps 1 > /dev/null 2>&1
wc -l gpurun_out/r1_side_kernels_ncu.csv
