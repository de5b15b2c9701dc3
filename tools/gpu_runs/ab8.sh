#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -3 > gpurun_out/pytest_gpu.log
timeout 150 python tools/ab_layout.py --mrl 520 >> gpurun_out/ab8.log 2>&1
timeout 240 python bench.py --steps 20 --warmup 4 --no-cpu --no-e2e > gpurun_out/bench_ab8.log 2>&1
