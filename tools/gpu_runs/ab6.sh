#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -15 > gpurun_out/pytest_gpu.log
for m in 520; do
LIFE_DEBUG=1 timeout 300 python tools/ab_layout.py --mrl $m >> gpurun_out/ab6.log 2>&1
LIFE_DEBUG=1 LIFE_B200_LIB=$PWD/build/p4/liblife_b200.so timeout 300 python tools/ab_layout.py --mrl $m >> gpurun_out/ab6.log 2>&1
done
