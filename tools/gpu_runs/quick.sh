#!/bin/bash
# quick check: GPU parity tests + one C2 bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -30 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-cpu > gpurun_out/bench_quick.log 2>&1
