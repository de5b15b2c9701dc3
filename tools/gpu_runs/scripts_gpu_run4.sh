#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^  " | tail -30 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 4 --no-cpu > gpurun_out/bench_c2_ws.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsc_ws -s 1 -c 1 -o gpurun_out/prof_dsc_ws python tools/prof_spmv.py --config c2 > gpurun_out/ncu_dsc_ws.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wc_ws -s 1 -c 1 -o gpurun_out/prof_wc_ws python tools/prof_spmv.py --config c2 > gpurun_out/ncu_wc_ws.log 2>&1
