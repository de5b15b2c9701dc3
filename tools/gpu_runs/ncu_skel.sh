#!/bin/bash
mkdir -p gpurun_out
LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsc_tc -s 15 -c 1 -o gpurun_out/tc_skel -f python tools/tc_isolate.py > gpurun_out/ncu_skel.log 2>&1
