#!/bin/bash
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_stream tools/ubench/tma_stream.cu && timeout 120 /tmp/tma_stream > gpurun_out/tma_stream.log 2>&1
