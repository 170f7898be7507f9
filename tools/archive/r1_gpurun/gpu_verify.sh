#!/bin/bash
# Re-entry check: build artefacts travel in-tree; full GPU suite + smoke + default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/verify_tests.log 2>&1; tail -3 gpurun_out/verify_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/verify_bench.jsonl 2> gpurun_out/verify_bench.err; tail -1 gpurun_out/verify_bench.jsonl
timeout 600 python bench.py --contraction ntt --no-cpu-baseline > gpurun_out/verify_bench_ntt.jsonl 2>> gpurun_out/verify_bench.err; tail -1 gpurun_out/verify_bench_ntt.jsonl
