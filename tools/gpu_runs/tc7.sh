#!/bin/bash
mkdir -p gpurun_out
LIFE_B200_LIB=$PWD/build/st3/liblife_b200.so timeout 600 python tools/tc_isolate.py > gpurun_out/tc_iso3.log 2>&1
