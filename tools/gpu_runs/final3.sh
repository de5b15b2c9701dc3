#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep_c5.py > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
timeout 600 python tools/sweep_c5.py --nnz 16e6,256e6 --skew zipf >> gpurun_out/sweep_c5.jsonl 2>> gpurun_out/sweep_c5.err
