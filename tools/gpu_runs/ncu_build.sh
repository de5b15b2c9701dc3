#!/bin/bash
mkdir -p gpurun_out
TC_FLAGS=0x7e LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsc_tc -s 5 -c 1 -o gpurun_out/tc_build -f python tools/tc_isolate.py > gpurun_out/ncu_build.log 2>&1
