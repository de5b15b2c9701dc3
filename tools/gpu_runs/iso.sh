#!/bin/bash
# producer/consumer isolation of the ws kernels at C2 (diagnostic build)
mkdir -p gpurun_out
WS_MODES=${WS_MODES:-0,1,2,0x101,0x401} LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so WS_PROD=8 timeout 900 python tools/ws_isolate.py > gpurun_out/iso.log 2>&1
