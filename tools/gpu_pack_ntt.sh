#!/bin/bash
mkdir -p gpurun_out

PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 256 2>&1 | tail -4
PYTHONPATH=. timeout 600 python tools/probe_pack_ntt.py 16 2>&1 | tail -4
