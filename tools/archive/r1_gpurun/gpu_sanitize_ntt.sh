#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck.log 2>&1; tail -2 gpurun_out/sanitizer_memcheck.log
timeout 900 $CS --tool racecheck python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck.log 2>&1; grep -E "RACECHECK SUMMARY|Race reported" gpurun_out/sanitizer_racecheck.log | sed 's/(CUtensorMap.*//' | head -6
timeout 900 $CS --tool synccheck python __graft_entry__.py smoke > gpurun_out/sanitizer_synccheck.log 2>&1; tail -1 gpurun_out/sanitizer_synccheck.log
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_ntt.py -x -q -k "TOY or over5 or transpose or refusal or adversarial" > gpurun_out/sanitizer_memcheck_ntt_tests.log 2>&1; tail -3 gpurun_out/sanitizer_memcheck_ntt_tests.log
