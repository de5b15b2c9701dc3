#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_wctc.json 2> gpurun_out/bench_wctc.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --layout fma > gpurun_out/bench_fma.json 2> gpurun_out/bench_fma.err
