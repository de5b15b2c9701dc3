#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --layout sparse > gpurun_out/qb_sparse.json 2> gpurun_out/qb.err
LIFE_B200_LIB=$PWD/build/spmv_ldg/liblife_b200.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --layout sparse > gpurun_out/qb_sparse_ldg.json 2>> gpurun_out/qb.err
timeout 1500 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/qb_c4.json 2>> gpurun_out/qb.err
