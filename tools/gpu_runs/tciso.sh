#!/bin/bash
# role isolation of the tensor-core DSC (diagnostic build: make -C paper_1905_06234_b200/csrc diag)
mkdir -p gpurun_out
TC_FLAGS=${TC_FLAGS:-0,4,1,2,0x6,0x7,0xff} LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so timeout 600 python tools/tc_isolate.py > gpurun_out/tc_iso.log 2>&1
