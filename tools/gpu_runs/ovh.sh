#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/solve_overhead.py > gpurun_out/solve_overhead.log 2>&1
