#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bal_on.json 2> gpurun_out/bal_on.err
LIFE_WS_ROUND_ROBIN=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bal_off.json 2> gpurun_out/bal_off.err
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
