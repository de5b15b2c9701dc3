#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep_c5.py --nnz 16e6,256e6 --skew zipf > gpurun_out/hot_zipf.jsonl 2> gpurun_out/hot.err
LIFE_WS_NO_HOT=1 timeout 600 python tools/sweep_c5.py --nnz 16e6,256e6 --skew zipf > gpurun_out/hot_zipf_off.jsonl 2>> gpurun_out/hot.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/qb.json 2>> gpurun_out/hot.err
