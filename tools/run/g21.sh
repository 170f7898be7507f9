set -x
timeout 900 python -m pytest tests/test_gpu_wire.py -q -x 2>&1 | tail -4
for v in "" "--wire" "" "--wire"; do timeout 300 python tools/probe.py --T 2048 --reps 60 $v | sed "s/^/[$v] /"; done
for v in "" "--wire"; do timeout 300 python tools/probe.py --d_out 16384 --d_in 2048 --T 255 --reps 40 $v | sed "s/^/[$v] /"; done
