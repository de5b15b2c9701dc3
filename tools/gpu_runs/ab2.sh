#!/bin/bash
mkdir -p gpurun_out
for m in 4 520; do
LIFE_DEBUG=1 timeout 300 python tools/ab_layout.py --mrl $m >> gpurun_out/ab2.log 2>&1
LIFE_DEBUG=1 LIFE_WS_UNSTAGED=1 timeout 300 python tools/ab_layout.py --mrl $m >> gpurun_out/ab2.log 2>&1
done
