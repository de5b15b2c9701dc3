#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --layout tensor > gpurun_out/t_def.json 2> gpurun_out/t.err
LIFE_B200_LIB=$PWD/build/g3u2/liblife_b200.so timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --layout tensor > gpurun_out/t_g3u2.json 2>> gpurun_out/t.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/qb.json 2>> gpurun_out/t.err
