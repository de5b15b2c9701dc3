#!/bin/bash
# tcgen05 descriptor / accuracy / throughput probe (tools/ubench/tc_probe.cu)
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tc_probe tools/ubench/tc_probe.cu && timeout 60 /tmp/tc_probe > gpurun_out/tc_probe.log 2>&1
echo rc=$? >> gpurun_out/tc_probe.log
