#!/bin/bash
# round-2 state check: GPU tests, default bench line, reference arm, random-access probes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
lscpu > gpurun_out/lscpu.txt 2>&1
WITH_REF=1 bash tools/gpu_runs/r02_tests.sh
timeout 300 tools/ubench/scatter_probe > gpurun_out/scatter_probe.log 2>&1
timeout 300 tools/ubench/gather_probe > gpurun_out/gather_probe.log 2>&1
tail -40 gpurun_out/scatter_probe.log gpurun_out/gather_probe.log
