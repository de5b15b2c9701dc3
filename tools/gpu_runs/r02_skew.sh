#!/bin/bash
# skew sweep (uniform vs Zipf fascicles vs one 5% voxel), then the GPU suite and bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python tools/bin_check.py --skew > gpurun_out/bin_skew.log 2>&1
cat gpurun_out/bin_skew.log
bash tools/gpu_runs/r02_tests.sh
