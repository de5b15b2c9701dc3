#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "solver_matches_reference" 2>&1 | grep -v "^  " | tail -60 > gpurun_out/pytest_solver.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsc_f32 -s 1 -c 1 -o gpurun_out/prof_dsc_v1 python tools/prof_spmv.py --config c2 > gpurun_out/ncu_dsc.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wc_f32 -s 1 -c 1 -o gpurun_out/prof_wc_v1 python tools/prof_spmv.py --config c2 > gpurun_out/ncu_wc.log 2>&1
