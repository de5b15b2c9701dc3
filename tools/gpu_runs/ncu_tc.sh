#!/bin/bash
# ncu --set full of one tensor-core DSC launch at C2
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsc_tc -s 1 -c 1 -o gpurun_out/tc_dsc -f python tools/prof_spmv.py --reps 2 --layout tensor > gpurun_out/ncu_tc.log 2>&1
