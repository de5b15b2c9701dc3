#!/bin/bash
# first GPU session: tests, smoke, bench
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 4 > gpurun_out/bench_c2.log 2>&1
