#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
