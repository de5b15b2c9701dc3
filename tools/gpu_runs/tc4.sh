#!/bin/bash
mkdir -p gpurun_out
export LIFE_DEBUG=1
timeout 300 python tools/tc_check.py > gpurun_out/tc_c2.log 2>&1
echo "rc=$?" >> gpurun_out/tc_c2.log
unset LIFE_DEBUG
LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so timeout 600 python tools/tc_isolate.py > gpurun_out/tc_iso.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsc_tc -s 1 -c 1 -o gpurun_out/tc_dsc -f python tools/prof_spmv.py --reps 2 > gpurun_out/ncu_tc.log 2>&1
