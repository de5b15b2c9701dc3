#!/bin/bash
# parity + staged vs unstaged A/B at C2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 4 --no-cpu --no-e2e > gpurun_out/bench_staged.log 2>&1
LIFE_WS_UNSTAGED=1 timeout 600 python bench.py --steps 20 --warmup 4 --no-cpu --no-e2e > gpurun_out/bench_unstaged.log 2>&1
