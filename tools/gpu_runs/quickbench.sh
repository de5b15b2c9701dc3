#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/qb.json 2> gpurun_out/qb.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --layout fma > gpurun_out/qb_fma.json 2>> gpurun_out/qb.err
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
