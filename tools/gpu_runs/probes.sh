#!/bin/bash
# random-access microbenchmarks (gathers / reductions, LSU vs TMA paths)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 tools/ubench/scatter_probe > gpurun_out/scatter_probe.log 2>&1
timeout 300 tools/ubench/gather_probe > gpurun_out/gather_probe.log 2>&1
cat gpurun_out/scatter_probe.log gpurun_out/gather_probe.log
