#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -30 > gpurun_out/pytest_gpu.log
