#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "rc=$?" >> gpurun_out/bench_c4.err
