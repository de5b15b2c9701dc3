#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -3 > gpurun_out/pytest_gpu.log
echo default >> gpurun_out/ab7.log; timeout 300 python tools/ab_layout.py --mrl 520 >> gpurun_out/ab7.log 2>&1
for v in p4 p8cp p4cp p4wc2; do
echo $v >> gpurun_out/ab7.log
LIFE_B200_LIB=$PWD/build/$v/liblife_b200.so timeout 300 python tools/ab_layout.py --mrl 520 >> gpurun_out/ab7.log 2>&1
done
