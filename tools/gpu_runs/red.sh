#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/red.json 2> gpurun_out/red.err
LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so WS_PROD=8 timeout 900 python tools/ws_isolate.py > gpurun_out/iso_red.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
