#!/bin/bash
mkdir -p gpurun_out
LIFE_B200_LIB=$PWD/build/cpasync/liblife_b200.so timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/cpa.json 2> gpurun_out/cpa.err
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/base.json 2> gpurun_out/base.err
