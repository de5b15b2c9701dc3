#!/bin/bash
# tensor-core vs CUDA-core DSC / WC: accuracy against the fp64 family and timing, C1 and C2
mkdir -p gpurun_out
export LIFE_DEBUG=1
timeout 120 python tools/tc_check.py --c1 > gpurun_out/tc_c1.log 2>&1
timeout 300 python tools/tc_check.py > gpurun_out/tc_c2.log 2>&1
unset LIFE_DEBUG
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
