#!/bin/bash
# round-2 final check, driver-like: build check, smoke, full GPU suite, bench (N=1), reference arm
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
WITH_REF=1 bash tools/gpu_runs/r02_tests.sh
