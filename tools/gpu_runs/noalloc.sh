#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/tc_check.py > gpurun_out/tc_c2.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --layout sparse > gpurun_out/qb_sparse.json 2> gpurun_out/qb.err
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/qb_c4.json 2>> gpurun_out/qb.err
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
