#!/bin/bash
# Experiment builds: libphe_<name>.so with extra -D flags (the probe selects one with PHE_LIB).
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC,-O2 \
  -I include "$@" -o paper_2505_07329_b200/libphe_$name.so paper_2505_07329_b200/csrc/*.cu
