#!/bin/bash
mkdir -p gpurun_out
cd tools/ubench && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2rand l2rand.cu && cd ../..
for nf in 500000 50000 8000; do timeout 300 /tmp/l2rand $nf; done > gpurun_out/l2rand.log 2>&1
